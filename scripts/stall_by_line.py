"""Map ncu SASS stall samples to CUDA source lines via nvdisasm line info.

    python scripts/stall_by_line.py <sass.csv from ncu --page source --print-source sass> <nvdisasm -g -c output> <mangled fn>
"""
import collections
import csv
import re
import sys

sass_csv, dis, fn = sys.argv[1:4]
rows = list(csv.reader(open(sass_csv)))
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows[2:] if len(r) > si]
start = int(data[0][0], 16)
samples = {int(r[0], 16) - start: int(r[si]) for r in data if r[si].isdigit()}
# nvdisasm: "//## File ..., line N" comments precede instructions
lines = open(dis).read().splitlines()
inside, cur, off2line = False, None, {}
for l in lines:
    if l.startswith(".text.") and fn in l:
        inside = True
        continue
    if inside and l.startswith(".text.") and fn not in l:
        break
    if not inside:
        continue
    m = re.search(r'line (\d+)', l)
    if l.strip().startswith("//##") and m:
        cur = int(m.group(1))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m:
        off2line[int(m.group(1), 16)] = cur
agg = collections.Counter()
for off, s in samples.items():
    agg[off2line.get(off)] += s
tot = sum(agg.values())
print("total samples", tot)
for ln, s in agg.most_common(40):
    print(f"{s:6d} {100 * s / tot:5.1f}%  line {ln}")
