"""Registers / spills per kernel from an `nvcc -Xptxas -v` log (stdin)."""
import re
import subprocess
import sys

cur = sp = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = cur.split("(")[0]
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        sp = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        if len(sys.argv) < 2 or re.search(sys.argv[1], cur):
            print(f"{cur:60s} regs {m.group(1):>4s} spill {sp}")
        cur = None
