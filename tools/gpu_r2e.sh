mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_fullsize_oracle.py -p no:cacheprovider 2>&1 | tail -30 > gpurun_out/gpu_tests_r2e.log
