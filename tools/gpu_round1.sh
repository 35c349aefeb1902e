# round-1 measurement batch (bench line, reference arm, kernel timings, launch list)
set -x
python bench.py --steps 20 --warmup 3 > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err; tail -3 gpurun_out/bench_r1b.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r1b.json 2>&1
python tools/prof_kernels.py 5 > gpurun_out/prof_kernels_r1b.txt 2>&1
python bench.py --steps 2 --warmup 3 --no-step --no-cpu > gpurun_out/plain_bench.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1b.csv python bench.py --steps 2 --warmup 3 --no-step --no-cpu > /dev/null 2>&1
cat gpurun_out/bench_r1b.json gpurun_out/bench_ref_r1b.json gpurun_out/prof_kernels_r1b.txt
