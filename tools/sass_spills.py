"""Spill (STL/LDL) instructions and total instruction counts per CUDA source line of a kernel in an object file.

    python tools/sass_spills.py obj.o kernel_substring [top]
"""
import collections
import re
import subprocess
import sys
import tempfile
import os

obj, pat = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cubin = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")][0]
out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
infn = False
line = None
spill = collections.Counter()
instr = collections.Counter()
for L in out.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", L)
    if m:
        infn = pat in m.group(1)
        continue
    if not infn:
        continue
    m = re.search(r'//## File ".*?([^/"]+)", line (\d+)(.*)', L)
    if m:
        line = (m.group(1), int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", L):
        instr[line] += 1
        if " STL" in L or " LDL" in L:
            spill[line] += 1
print("instructions", sum(instr.values()), "spill instr", sum(spill.values()))
for k, v in spill.most_common(top):
    print(f"{v:6d} spill  {instr[k]:7d} instr  {k[0]}:{k[1]}")
