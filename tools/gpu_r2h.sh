mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rect_path.py -q -x -p no:cacheprovider 2>&1 | tail -3 > gpurun_out/rect_tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize_oracle.py -q -s -k "config3_pmg or config1" -p no:cacheprovider 2>&1 | tail -4 >> gpurun_out/rect_tests.log
timeout 600 python tools/time_rect.py 2 4 5 > gpurun_out/time_rect.log 2>&1
