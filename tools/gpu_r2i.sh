mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_fullsize_oracle.py -q -s -p no:cacheprovider 2>&1 | grep -E "config|Jv|48|passed|failed|Error|assert" | tail -30 > gpurun_out/fullsize_r2i.log
