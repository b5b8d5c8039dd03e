"""Attribute an ncu SASS source-page CSV (executed instructions, stall samples) to
CUDA source lines via nvdisasm -g line info of the same cubin.
usage: sass_lines.py <sass.csv> <nvdisasm -g -c output> <mangled kernel name> [topN]"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
ie, ws = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
base = int(data[0][0], 16)
txt = open(sys.argv[2]).read().split("\n")
kname = sys.argv[3]
line_of = {}
cur = None
inside = False
for t in txt:
    if t.startswith("//----") and ".text." in t:
        inside = kname in t
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', t)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", t)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
inst = defaultdict(float)
stall = defaultdict(float)
for r in data:
    off = int(r[0], 16) - base
    k = line_of.get(off, ("?", 0))
    inst[k] += float(r[ie] or 0)
    stall[k] += float(r[ws] or 0)
ti, ts = sum(inst.values()), sum(stall.values())
src = {}
for k in sorted(inst, key=lambda k: -inst[k])[: int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{k[0]}:{k[1]:<5} inst {inst[k] / ti * 100:5.1f}%  stall {stall[k] / ts * 100:5.1f}%")
