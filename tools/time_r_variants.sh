# A/B of build variants on R / Jv at config 2 (each variant in its own process)
for v in libpmgflow_b200.so libpmgflow_b200_v64.so libpmgflow_b200_v32.so; do
  echo "== $v"; PMGB_LIB=$PWD/paper_2202_09733_b200/$v python tools/time_residual.py 2 20
  PMGB_LIB=$PWD/paper_2202_09733_b200/$v python tools/time_residual.py 1 50
done
