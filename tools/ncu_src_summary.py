"""Summarise an `ncu --page source --csv --print-source sass` export:
stall reasons by total samples, top instructions, opcode mix."""
import csv
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[2:] if len(r) == len(hdr) and r[0].startswith("0x")]
f = lambda r, k: float(r[ix[k]] or 0)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
for r in data:
    for s in stalls:
        tot[s] += f(r, s)
T = sum(tot.values())
print(f"samples {T:.0f}")
for s, v in tot.most_common(10):
    print(f"  {s:26s} {100 * v / T:5.1f}%")
ops = Counter()
inst = Counter()
for r in data:
    op = r[ix["Source"]].strip().split()[0] if r[ix["Source"]].strip() else "?"
    if op.startswith("@"):
        op = r[ix["Source"]].strip().split()[1]
    op = op.split(".")[0]
    ops[op] += f(r, "Warp Stall Sampling (All Samples)")
    inst[op] += f(r, "Instructions Executed")
I = sum(inst.values())
print(f"warp instructions executed {I:.3g}")
for op, v in inst.most_common(14):
    print(f"  {op:10s} inst {100 * v / I:5.1f}%   stall-samples {100 * ops[op] / T:5.1f}%")
print("top stalled instructions:")
top = sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]
for r in top:
    main = max(stalls, key=lambda s: f(r, s))
    print(f"  {f(r, 'Warp Stall Sampling (All Samples)'):7.0f} {main:22s} {r[ix['Source']].strip()[:70]}")
