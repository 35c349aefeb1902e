# ncu capture of the three R kernels at config 2; export summaries on the box
python tools/time_residual.py 2 1 > gpurun_out/plain_r.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"k_assemble|k_fvn|k_trace" -c 3 -o /tmp/prof_r python tools/time_residual.py 2 1 > /dev/null 2>&1
ncu -i /tmp/prof_r.ncu-rep --page raw --csv > gpurun_out/ncu_r_raw.csv 2>/dev/null
ncu -i /tmp/prof_r.ncu-rep --page details --csv > gpurun_out/ncu_r_details.csv 2>/dev/null
for k in k_assemble k_fvn k_trace; do
  ncu -i /tmp/prof_r.ncu-rep -k regex:$k --page source --csv --print-source sass > gpurun_out/ncu_r_src_$k.csv 2>/dev/null
done
ls -la gpurun_out
