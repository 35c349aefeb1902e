# ncu of the Jv chain of the rectangle path (config 2): durations only
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k regex:"k_r(face|grad|asm|fc)" -c 40 --csv python tools/time_residual.py ${1:-2} 2 > gpurun_out/ncu_rect_jv.csv 2>/dev/null
