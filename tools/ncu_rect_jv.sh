# ncu capture of the Jv chain of the rectangle path (config 2): full set, source-level stall summaries
mkdir -p gpurun_out
ncu -f --set full --clock-control none --import-source on -k regex:"k_r(gf|asm)" --launch-skip 10 -c 2 -o /tmp/prof_rect_jv python tools/time_residual.py ${1:-2} 1 > gpurun_out/ncu_rect_jv_run.log 2>&1
ncu -i /tmp/prof_rect_jv.ncu-rep --page details --csv > gpurun_out/ncu_rect_jv_details.csv 2>/dev/null
for k in k_rgf k_rasm; do
  ncu -i /tmp/prof_rect_jv.ncu-rep -k regex:$k -c 1 --page source --csv --print-source sass > /tmp/ncu_rect_jv_src_$k.csv 2>/dev/null
  python tools/ncu_src_summary.py /tmp/ncu_rect_jv_src_$k.csv > gpurun_out/ncu_src_jv_$k.txt 2>&1
done
ls -la gpurun_out | head
