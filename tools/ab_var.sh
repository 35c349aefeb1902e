#!/bin/bash
# A/B of experiment builds (tools/build_variant.sh) on the rect path, interleaved twice:
#   tools/ab_var.sh "<configs>" name1 name2 ...
mkdir -p gpurun_out
cfgs=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    echo "== $v" | tee -a gpurun_out/ab_var.log
    PMGB_LIB=$PWD/paper_2202_09733_b200/libpmgflow_b200_$v.so RECT_PATHS=${RECT_PATHS:-rect} python tools/time_rect.py $cfgs 2>&1 | \
      python -c "
import sys, json
for l in sys.stdin:
    try: d = json.loads(l)
    except Exception: print(l.rstrip()); continue
    print(' '.join([f\"c{d['config']}\"] + [f\"{k}: R {v['r_us']:.1f} Jv {v['jv_us']:.1f} stageJv {v.get('stage_jv_us', 0):.1f} defect {v.get('defect_us', 0):.1f}\" for k, v in d.items() if isinstance(v, dict)]))
" | tee -a gpurun_out/ab_var.log
  done
done
