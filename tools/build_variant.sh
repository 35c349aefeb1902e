#!/bin/bash
# Experiment build of the rectangle kernels only: tools/build_variant.sh <name> [-DMACRO=..]...
# compiles csrc/fr_rect.cu (config-2 / config-4 instances only, -DPMGB_RECT_DEV; FULL=1: every instance) with the
# given defines and links it with the default build's other objects into
# paper_2202_09733_b200/libpmgflow_b200_<name>.so (load with PMGB_LIB=...).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
C=paper_2202_09733_b200/csrc
mkdir -p $C/build_var
DEV=-DPMGB_RECT_DEV; [ -n "$FULL" ] && DEV=
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
  --fmad=true $DEV "$@" -Xptxas -v -c $C/fr_rect.cu -o $C/build_var/fr_rect_$name.o 2> $C/build_var/fr_rect_$name.log
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2202_09733_b200/libpmgflow_b200_$name.so \
  $C/build_var/fr_rect_$name.o $C/build/fr_kernels.o $C/build/fr_mixed.o $C/build/ej_kernels.o $C/build/krylov_kernels.o $C/build/capi.o -lcudart
echo built libpmgflow_b200_$name.so
