"""profiles/traffic_r2.json from an ncu raw CSV of one R chain at config 2
(tools/ncu_rect.sh): DRAM bytes read + written per kernel of the first
chain, their sum (bench.py's roofline.traffic) and the hash of the CUDA
sources the capture was made with (bench.py marks a stale figure).

    python tools/traffic_stamp.py gpurun_out/ncu_rect_raw.csv
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import src_hash  # noqa: E402

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
units = rows[1]
chain, seen = {}, set()
for r in rows[2:]:
    name = r[ix["Kernel Name"]].split("(")[0]
    if name in seen:
        break
    seen.add(name)

    def mb(key):
        v = float(r[ix[key]])
        u = units[ix[key]]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    chain[name] = {"dram_read_bytes": mb("dram__bytes_read.sum"), "dram_write_bytes": mb("dram__bytes_write.sum"),
                   "duration_us": float(r[ix["gpu__time_duration.sum"]]) / (1e3 if units[ix["gpu__time_duration.sum"]] == "nsecond" else 1)}
tot = sum(v["dram_read_bytes"] + v["dram_write_bytes"] for v in chain.values())
out = {"config2_R_bytes": tot, "compulsory_bytes": 16 * 6553600, "ratio": tot / (16 * 6553600),
       "per_kernel": chain, "src_hash": src_hash(),
       "source": "ncu --set full, tools/ncu_rect.sh (one R chain at config 2, serialised launches)"}
(ROOT / "profiles" / "traffic_r2.json").write_text(json.dumps(out, indent=1) + "\n")
print(json.dumps(out, indent=1))
