#!/bin/bash
for rep in 1 2; do
  for lib in libpmgflow_b200.so libv_p3.so; do
    for k in 4 1; do
      echo -n "$lib "; PMGB_LIB=$PWD/paper_2202_09733_b200/$lib python tools/time_residual.py $k 100 2>/dev/null | tr '\n' ' '; echo
    done
  done
done
