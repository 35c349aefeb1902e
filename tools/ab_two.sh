#!/bin/bash
# A/B of two library builds on R / Jv at configs 2 and 4: tools/ab_two.sh libA.so libB.so
for rep in 1 2; do
  for lib in "$@"; do
    for k in 2 4; do
      echo -n "$lib "; PMGB_LIB=$PWD/paper_2202_09733_b200/$lib python tools/time_residual.py $k 100 2>/dev/null | tr '\n' ' '; echo
    done
  done
done
