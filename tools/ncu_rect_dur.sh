# durations / DRAM bytes of one rect R chain + one Jv chain at a config (ncu, serialised)
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_r(face|grad|asm|fc|gf)" -c 24 --csv python tools/time_residual.py ${1:-2} 2 > gpurun_out/ncu_rect_dur.csv 2>/dev/null
python - <<'PY'
import csv
from collections import defaultdict
rows=[r for r in csv.reader(open('gpurun_out/ncu_rect_dur.csv')) if len(r)>10]
hdr=rows[0]; ix={h:i for i,h in enumerate(hdr)}
agg=defaultdict(dict)
for r in rows[1:]:
    if not r[ix['ID']].isdigit(): continue
    agg[(int(r[ix['ID']]), r[ix['Kernel Name']].split('(')[0])][r[ix['Metric Name']]]=r[ix['Metric Value']]
with open('gpurun_out/ncu_rect_dur.txt','w') as f:
    for (i,k),v in sorted(agg.items()):
        f.write(f"{i:3d} {k:32s} {float(v['gpu__time_duration.sum'])/1e3:8.1f} us  rd {float(v['dram__bytes_read.sum'])/1e6:7.1f} MB  wr {float(v['dram__bytes_write.sum'])/1e6:7.1f} MB  inst {float(v['smsp__inst_executed.sum'])/1e6:6.2f} M  warps {v['sm__warps_active.avg.pct_of_peak_sustained_active']}\n")
PY
