#!/bin/bash
# Round validation on the GPU box: every GPU test, smoke(), both bench arms, the ncu
# launch list of the bench command and one full ncu capture of the R / Jv chains at
# config 2 (DRAM traffic stamped into profiles/traffic_r2.json).
#   gpurun --timeout 3600 -- 'bash tools/validate_round.sh r2x'   -> gpurun_out/*_r2x.*
tag=${1:-r2x}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
( time timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider ) > gpurun_out/gpu_suite_$tag.log 2>&1; tail -4 gpurun_out/gpu_suite_$tag.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2 | tee gpurun_out/smoke_$tag.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$tag.json 2> gpurun_out/bench_ref_$tag.err; tail -c 600 gpurun_out/bench_ref_$tag.json
python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; tail -c 2500 gpurun_out/bench_$tag.json
FLAGS="--steps 2 --warmup 3 --no-step --no-cpu --no-configs --no-mbnk"
python bench.py $FLAGS > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$tag.csv python bench.py $FLAGS > /dev/null 2>&1
python - $tag "$FLAGS" <<'PY'
import csv, sys
from collections import defaultdict
tag, flags = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(f"gpurun_out/launches_{tag}.csv")) if len(r) > 10]
ix = {h: i for i, h in enumerate(rows[0])}
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[ix["ID"]].isdigit():
        a = agg[r[ix["Kernel Name"]].split("(")[0]]
        a[0] += 1
        a[1] += float(r[ix["Metric Value"]].replace(",", "")) / 1e3
tot = sum(v[1] for v in agg.values())
with open(f"gpurun_out/launches_{tag}.txt", "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none -c 400: bench.py {flags} (serialised, cold-cache per launch)\n")
    f.write(f"total {tot:.1f} us over {sum(v[0] for v in agg.values())} launches\n")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        f.write(f"{v[1]:10.1f} us {100 * v[1] / tot:5.1f}%  n={v[0]:4d}  {k}\n")
print(open(f"gpurun_out/launches_{tag}.txt").read())
PY
rm -f gpurun_out/launches_$tag.csv
bash tools/ncu_rect.sh 2 > /dev/null 2>&1
python tools/traffic_stamp.py gpurun_out/ncu_rect_raw.csv > gpurun_out/traffic_$tag.json 2>&1; head -8 gpurun_out/traffic_$tag.json
cp profiles/traffic_r2.json gpurun_out/traffic_r2.json
for k in k_rgf k_rasm; do python tools/ncu_src_summary.py gpurun_out/ncu_rect_src_$k.csv > gpurun_out/ncu_src_${k}_$tag.txt 2>&1; done
mv gpurun_out/ncu_rect_details.csv gpurun_out/ncu_rect_details_$tag.csv
rm -f gpurun_out/ncu_rect_raw.csv gpurun_out/ncu_rect_src_*.csv gpurun_out/*.ncu-rep
ls -la gpurun_out
