# round-2 validation: full GPU suite, smoke, bench, launch list, traffic capture
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/gpu_suite_r2k.log; cat gpurun_out/gpu_suite_r2k.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r2k.log 2>&1; tail -2 gpurun_out/smoke_r2k.log
timeout 900 python bench.py > gpurun_out/bench_r2k.json 2> gpurun_out/bench_r2k.err; tail -c 600 gpurun_out/bench_r2k.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r2k.json 2>&1; tail -c 400 gpurun_out/bench_ref_r2k.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r2k.csv python bench.py --steps 2 --warmup 3 --no-step --no-cpu --no-configs --no-mbnk > gpurun_out/ncu_launch_r2k.log 2>&1
bash tools/ncu_rect.sh 2
