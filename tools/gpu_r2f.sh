mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_solver.py tests/test_gpu_partitioned_solver.py tests/test_gpu_rect_path.py -q -x -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/gpu_tests_r2f.log
