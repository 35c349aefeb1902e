#!/bin/bash
# Config-5 physics (vortex array, p{5-4}, ESDIRK3 at CFL 100): which smoother pairs converge
# as the mesh goes 512^2 -> 1024^2.   tools/c5_explore.sh NX NSTEPS PREC VARIANT...
nx=$1; ns=$2; prec=$3; shift 3
mkdir -p gpurun_out
for v in "$@"; do
  NX=$nx BLOCK_PRECISION=$prec MAX_PTC=${MAX_PTC:-12} timeout ${TMO:-900} python tools/solver_steps.py 5 $ns "$v" 2>&1 | cut -c1-1500 | tee -a gpurun_out/c5_explore_${nx}.log
done
