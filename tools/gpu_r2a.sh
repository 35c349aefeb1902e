set -x
mkdir -p gpurun_out
nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
tools/bin/dmma_probe > gpurun_out/dmma_probe.jsonl 2>&1; cat gpurun_out/dmma_probe.jsonl
timeout 1500 python -m pytest tests/test_gpu_fullsize_oracle.py -x -q -s -m gpu 2>&1 | tail -30 > gpurun_out/fullsize_oracle.log; cat gpurun_out/fullsize_oracle.log
