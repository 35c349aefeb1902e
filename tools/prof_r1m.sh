# R kernels after the epilogue specialization: ncu --set full of one R at config 2 + bench launch list
python tools/time_residual.py 2 1 > gpurun_out/plain_r.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"k_assemble|k_fvn|k_trace" -c 3 -o /tmp/prof_r python tools/time_residual.py 2 1 > /dev/null 2>&1
ncu -i /tmp/prof_r.ncu-rep --page details --csv > gpurun_out/ncu_r_details_r1m.csv 2>/dev/null
ncu -i /tmp/prof_r.ncu-rep --page raw --csv > gpurun_out/ncu_r_raw_r1m.csv 2>/dev/null
python bench.py --steps 2 --warmup 3 --no-step --no-cpu --no-configs --no-mbnk > gpurun_out/plain_bench_r1m.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r1m.csv \
  python bench.py --steps 2 --warmup 3 --no-step --no-cpu --no-configs --no-mbnk > /dev/null 2>&1
