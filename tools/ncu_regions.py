"""Group an ncu SASS source export into runs of equal execution count and
print the heaviest runs with their opcode mix (where the instructions go)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
seen, uniq = set(), []
for r in rows[2:]:
    if len(r) == len(hdr) and r[0].startswith("0x") and r[0] not in seen:
        seen.add(r[0])
        uniq.append(r)
cnt = [(r[0], float(r[ix["Instructions Executed"]] or 0), r[1].strip()) for r in uniq]
tot = sum(c for _, c, _ in cnt)
runs, prev, ops, start = [], None, [], None
for a, c, src in cnt:
    if c != prev:
        if prev is not None:
            runs.append((prev, start, ops))
        prev, start, ops = c, a, []
    tok = src.split()
    ops.append((tok[1] if tok and tok[0].startswith("@") else (tok[0] if tok else "?")))
runs.append((prev, start, ops))
print(f"total warp-instr {tot:.4g}")
for c, a, o in sorted(runs, key=lambda x: -x[0] * len(x[2]))[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    mix = Counter(x.split(".")[0] for x in o).most_common(7)
    print(f"{100 * c * len(o) / tot:5.1f}%  exec {c:9.0f} x {len(o):4d}  {a[-5:]}  {mix}")
