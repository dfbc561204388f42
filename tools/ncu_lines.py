"""Stall samples per CUDA source line from an ncu report (--import-source on).

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import collections
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source=cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
cur = None
cur_line = None
tot = collections.Counter()
text = {}
total = 0
for L in out.split("\n"):
    if L.startswith('"File Path"'):
        cur = L.split(",", 1)[1].strip('"').split("/")[-1]
        continue
    m = re.match(r'^"(\d+)","(.*?)","-","-","(\d+)"', L)
    if m:  # CUDA source line row: its sample count is the sum over its SASS
        k = (cur, int(m.group(1)))
        tot[k] += int(m.group(3))
        text[k] = m.group(2)[:80]
        total += int(m.group(3))
print(f"total samples {total}")
for k, v in tot.most_common(top):
    print(f"{v:8d} {100 * v / total:5.1f}%  {k[0]}:{k[1]}  {text[k]}")
