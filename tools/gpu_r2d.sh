mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rect_path.py -q -x 2>&1 | tail -5 > gpurun_out/rect_tests.log
timeout 1200 python bench.py > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err
bash tools/ncu_rect.sh 2
python tools/traffic_stamp.py gpurun_out/ncu_rect_raw.csv > /dev/null && cp profiles/traffic_r2.json gpurun_out/
