#!/bin/bash
# A/B timing of library variants: tools/ab_libs.sh lib1.so lib2.so ...
# (bench.py R/Jv only, interleaved twice; prints value GDoF/s, R ms, Jv ms)
for rep in 1 2; do
  for lib in "$@"; do
    PMGB_LIB=$PWD/paper_2202_09733_b200/$lib python bench.py --no-step --no-configs --no-mbnk --no-cpu --steps 100 \
      > gpurun_out/ab_$lib.json 2>/dev/null
    python -c "import json,sys;d=json.load(open('gpurun_out/ab_$lib.json'));print('$lib', round(d['value'],3), round(d['ms_per_step']*1e3,1), round(d['jv_ms']*1e3,1))"
  done
done
