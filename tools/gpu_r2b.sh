mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_fullsize_oracle.py -q -s -m gpu 2>&1 | tail -40 > gpurun_out/fullsize_oracle_b.log
