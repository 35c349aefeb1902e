mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rect_path.py -q -x 2>&1 | tail -40 > gpurun_out/rect_tests.log
timeout 600 python tools/time_rect.py 2 4 3 > gpurun_out/time_rect.log 2>&1
