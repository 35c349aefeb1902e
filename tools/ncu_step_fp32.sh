python tools/step_profile.py 2 --fp32 --case-scheme > gpurun_out/step_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/step_launches.csv python tools/step_profile.py 2 --no-warm --fp32 --case-scheme > /dev/null 2>&1
python - <<'PY'
import csv
from collections import defaultdict
rows = list(csv.reader(open("gpurun_out/step_launches.csv")))
hdr = None; agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); name = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[name][0] += 1; agg[name][1] += float(d["Metric Value"].replace(",", "")) / 1e3
tot = sum(v[1] for v in agg.values())
with open("gpurun_out/step_breakdown.txt", "w") as f:
    f.write(f"total device time {tot / 1e3:.1f} ms over {sum(v[0] for v in agg.values())} launches\n")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{t / 1e3:9.2f} ms {100 * t / tot:5.1f}%  n={n:6d}  {k}\n")
PY
cat gpurun_out/step_plain.log gpurun_out/step_breakdown.txt
