"""Stall samples along the SASS of an `ncu --page source --csv --print-source sass`
export, in equal instruction-count segments (the kernels are straight-line,
so position = phase): per segment the share of samples, the top stall
reasons and the opcode mix."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
seen, data = set(), []
for r in rows[2:]:
    if len(r) == len(hdr) and r[0].startswith("0x") and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
nseg = int(sys.argv[2]) if len(sys.argv) > 2 else 16
f = lambda r, k: float(r[ix[k]] or 0)
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
T = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
n = len(data)
print(f"{n} instructions, {T:.0f} samples")
for s in range(nseg):
    seg = data[s * n // nseg:(s + 1) * n // nseg]
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in seg)
    c = Counter()
    ops = Counter()
    for r in seg:
        for st in stalls:
            c[st[6:]] += f(r, st)
        tok = r[ix["Source"]].split()
        ops[(tok[1] if tok[0].startswith("@") else tok[0]).split(".")[0]] += 1
    top = " ".join(f"{k}:{100 * v / max(tot, 1):.0f}" for k, v in c.most_common(4))
    mix = " ".join(f"{k}{v}" for k, v in ops.most_common(5))
    print(f"seg {s:2d} [{s * n // nseg:5d}] {100 * tot / T:5.1f}%  {top:60s} {mix}")
