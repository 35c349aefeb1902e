"""Registers / spills per kernel from an nvcc -Xptxas -v log (demangled)."""
import re, subprocess, sys
log = open(sys.argv[1]).read().splitlines()
pat = sys.argv[2] if len(sys.argv) > 2 else ""
cur = None
spill = ""
for line in log:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
    if "spill" in line:
        spill = line.strip()
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        name = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
        if pat in name:
            print(f"{m2.group(1):>4} regs  {spill[:60]:60s} {name[:80]}")
