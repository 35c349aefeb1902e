# round-1 (session 3) profile batch: bench launch list, R kernels + EJ apply ncu --set full
set -x
python bench.py --steps 2 --warmup 3 --no-step --no-cpu > gpurun_out/plain_bench_r1j.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r1j.csv \
  python bench.py --steps 2 --warmup 3 --no-step --no-cpu > /dev/null 2>&1
python tools/time_residual.py 2 1 > gpurun_out/plain_r.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"k_assemble|k_fvn|k_trace" -c 3 -o /tmp/prof_r python tools/time_residual.py 2 1 > /dev/null 2>&1
ncu -i /tmp/prof_r.ncu-rep --page details --csv > gpurun_out/ncu_r_details_r1j.csv 2>/dev/null
ncu -i /tmp/prof_r.ncu-rep --page raw --csv > gpurun_out/ncu_r_raw_r1j.csv 2>/dev/null
python tools/time_ej.py 256 20 > gpurun_out/time_ej_r1j.json 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"k_block_gemv" -c 2 -o /tmp/prof_ej python tools/time_ej.py 128 1 > /dev/null 2>&1
ncu -i /tmp/prof_ej.ncu-rep --page details --csv > gpurun_out/ncu_ej_details_r1j.csv 2>/dev/null
ncu -i /tmp/prof_ej.ncu-rep --page raw --csv > gpurun_out/ncu_ej_raw_r1j.csv 2>/dev/null
ls -la gpurun_out
