mkdir -p gpurun_out
python tools/prof_gj.py 64 2 > gpurun_out/gj_time2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_solver.py tests/test_gpu_mbnk.py -q -x -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/gj_tests.log
