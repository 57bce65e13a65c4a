"""Executed warp-instructions per CUDA source line from ncu's SASS source page + nvdisasm -g.

    python scripts/inst_by_line.py <sass.csv> <nvdisasm -g -c output> <mangled fn> [top]
"""
import collections
import csv
import re
import sys

sass_csv, dis, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 20
rows = list(csv.reader(open(sass_csv)))
h = rows[1]
ie = h.index("Instructions Executed")
data = [r for r in rows[2:] if len(r) > ie]
start = int(data[0][0], 16)
lines = open(dis).read().splitlines()
inside, cur, file_, off2line = False, None, "", {}
for l in lines:
    if l.startswith(".text.") and fn in l:
        inside = True
        continue
    if inside and l.startswith(".text.") and fn not in l:
        break
    if not inside:
        continue
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if l.strip().startswith("//##") and m:
        file_, cur = m.group(1).split("/")[-1], int(m.group(2))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m:
        off2line[int(m.group(1), 16)] = f"{file_}:{cur}"
agg = collections.Counter()
for r in data:
    if r[ie].isdigit():
        agg[off2line.get(int(r[0], 16) - start)] += int(r[ie])
tot = sum(agg.values())
print("total warp-instructions", tot)
for ln, s in agg.most_common(top):
    print(f"{s:12d} {100 * s / tot:5.1f}%  {ln}")
