#!/bin/bash
# A/B of the R-only k_assemble_async instantiation (PMGB_R_ONLY, register targets)
for rep in 1 2 3; do
  for v in "off:libpmgflow_b200.so:0" "r72:libpmgflow_b200.so:1" "r80:libv_r80.so:1" "r64:libv_r64.so:1"; do
    IFS=: read name lib on <<< "$v"
    PMGB_R_ONLY=$on PMGB_LIB=$PWD/paper_2202_09733_b200/$lib python bench.py --no-step --no-configs --no-mbnk --no-cpu \
      --steps 100 > gpurun_out/ab_$name.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_$name.json'));print('$name', round(d['value'],3), round(d['ms_per_step']*1e3,1), round(d['jv_ms']*1e3,1))"
  done
done
