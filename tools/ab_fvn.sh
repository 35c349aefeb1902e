#!/bin/bash
# A/B of the k_fvn register target (64 default vs 56 = 9 CTAs/SM) on R / Jv at configs 2 (p=4) and 4 (p=3)
for rep in 1 2; do
  for lib in libpmgflow_b200.so libv_f56.so; do
    for k in 2 4; do
      echo -n "$lib "; PMGB_LIB=$PWD/paper_2202_09733_b200/$lib python tools/time_residual.py $k 100 2>/dev/null | tr '\n' ' '; echo
    done
  done
done
