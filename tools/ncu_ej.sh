python tools/prof_gj.py 16 1 > gpurun_out/plain_gj.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"k_gj|k_blocks" -c 2 -o /tmp/prof_gj python tools/prof_gj.py 16 1 > /dev/null 2>&1
ncu -i /tmp/prof_gj.ncu-rep --page details --csv > gpurun_out/ncu_gj_details.csv 2>/dev/null
ncu -i /tmp/prof_gj.ncu-rep -k regex:k_gj --page source --csv --print-source sass > gpurun_out/ncu_gj_src.csv 2>/dev/null
ncu -i /tmp/prof_gj.ncu-rep -k regex:k_blocks --page source --csv --print-source sass > gpurun_out/ncu_blocks_src.csv 2>/dev/null
cat gpurun_out/plain_gj.log
