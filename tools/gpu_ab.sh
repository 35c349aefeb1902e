# A/B two library builds on the rect path: tools/gpu_ab.sh <lib_a> <lib_b> [configs]
mkdir -p gpurun_out
for lib in "$1" "$2"; do
  echo "== $lib" >> gpurun_out/ab.log
  PMGB_LIB=paper_2202_09733_b200/$lib python tools/time_rect.py ${3:-2} >> gpurun_out/ab.log 2>&1
done
