"""Per-instruction L1 shared-memory wavefronts from an ncu source export:
which loads/stores consume L1 bandwidth, and how much is bank-conflict
excess.  usage: ncu_l1.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
seen = set()
data = []
for r in rows[2:]:
    if len(r) == len(hdr) and r[0].startswith("0x") and r[ix["Address"]] not in seen:
        seen.add(r[ix["Address"]])
        data.append(r)
f = lambda r, k: float(r[ix[k]] or 0)
W = sum(f(r, "L1 Wavefronts Shared") for r in data)
X = sum(f(r, "L1 Wavefronts Shared Excessive") for r in data)
G = sum(f(r, "L1 Tag Requests Global") for r in data)
print(f"shared wavefronts {W:.3g}  excessive {X:.3g} ({100*X/max(W,1):.1f}%)  global tag requests {G:.3g}")
key = "L1 Wavefronts Shared Excessive" if "--excess" in sys.argv else "L1 Wavefronts Shared"
top = sorted(data, key=lambda r: -f(r, key))[:int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 25]
for r in top:
    print(f"  {f(r,'L1 Wavefronts Shared'):10.0f} ideal {f(r,'L1 Wavefronts Shared Ideal'):10.0f} exec {f(r,'Instructions Executed'):8.0f}  {r[ix['Address']]} {r[ix['Source']].strip()[:60]}")
