# ncu --set full of k_gj_inverse<100> (config-2 fine-level FD blocks, 64^2 mesh) + the DMMA/DFMA probe
mkdir -p gpurun_out
python tools/prof_gj.py 64 2 > gpurun_out/gj_time.log 2>&1
ncu -f --set full --clock-control none --import-source on -k regex:"k_gj_inverse" -c 1 -o /tmp/prof_gj python tools/prof_gj.py 64 1 > /dev/null 2>&1
ncu -i /tmp/prof_gj.ncu-rep --page details --csv > gpurun_out/ncu_gj_details.csv 2>/dev/null
ncu -i /tmp/prof_gj.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_gj_src.csv 2>/dev/null
ncu -i /tmp/prof_gj.ncu-rep --page raw --csv > gpurun_out/ncu_gj_raw.csv 2>/dev/null
