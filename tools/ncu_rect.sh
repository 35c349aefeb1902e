# ncu capture of the three rectangle-path R kernels at config 2 (R and Jv)
mkdir -p gpurun_out
python tools/time_residual.py ${1:-2} 1 > gpurun_out/plain_rect.log 2>&1 && \
ncu -f --set full --clock-control none --import-source on -k regex:"k_r(face|grad|asm|fc|gf)" -c 8 -o /tmp/prof_rect python tools/time_residual.py ${1:-2} 1 > gpurun_out/ncu_rect_run.log 2>&1
ncu -i /tmp/prof_rect.ncu-rep --page raw --csv > gpurun_out/ncu_rect_raw.csv 2>/dev/null
ncu -i /tmp/prof_rect.ncu-rep --page details --csv > gpurun_out/ncu_rect_details.csv 2>/dev/null
for k in k_rface k_rgrad k_rasm k_rfc k_rgf; do
  ncu -i /tmp/prof_rect.ncu-rep -k regex:$k -c 1 --page source --csv --print-source sass > gpurun_out/ncu_rect_src_$k.csv 2>/dev/null
done
# the .ncu-rep stays on the box (gpurun_out/ is capped at 64 MiB)
ls -la gpurun_out
