#!/bin/bash
# A/B of the compile-time epilogue instantiations of k_assemble_async:
# runtime switch (PMGB_EPI_SPECIALIZE=0) vs specialized (register targets
# R 72 / others 80 = default lib, others 72 = libv_k72.so); R and Jv at config 2,
# then one config-2 ESDIRK3 step (fp32 blocks) per variant
for rep in 1 2; do
  for v in "generic:libpmgflow_b200.so:0" "spec:libpmgflow_b200.so:1" "spec_k72:libv_k72.so:1"; do
    IFS=: read name lib on <<< "$v"
    PMGB_EPI_SPECIALIZE=$on PMGB_LIB=$PWD/paper_2202_09733_b200/$lib python bench.py --no-step --no-configs --no-mbnk \
      --no-cpu --steps 100 > gpurun_out/ab_$name.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/ab_$name.json'));print('$name', round(d['value'],3), round(d['ms_per_step']*1e3,1), round(d['jv_ms']*1e3,1))"
  done
done
for v in "generic:libpmgflow_b200.so:0" "spec:libpmgflow_b200.so:1" "spec_k72:libv_k72.so:1"; do
  IFS=: read name lib on <<< "$v"
  echo "== step $name"
  PMGB_EPI_SPECIALIZE=$on PMGB_LIB=$PWD/paper_2202_09733_b200/$lib BLOCK_PRECISION=fp32 python tools/solver_steps.py 2 1 esdirk3:ej-ej:5000 2>/dev/null | tail -1 | cut -c1-300
done
