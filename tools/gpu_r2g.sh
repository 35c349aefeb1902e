mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_dropin_reference.py -q -x -p no:cacheprovider 2>&1 | tail -25 > gpurun_out/dropin.log
