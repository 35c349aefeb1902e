# A/B of build variants on R / Jv at config 2 (each variant in its own process)
for v in "$@"; do
  echo "== $v"; PMGB_LIB=$PWD/paper_2202_09733_b200/$v python tools/time_residual.py 2 20
done
