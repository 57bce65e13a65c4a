"""Per-source-line stall-reason breakdown (top lines) from ncu's SASS source page + nvdisasm -g.

    python scripts/stall_reasons_by_line.py <sass.csv> <nvdisasm -g -c output> <mangled fn> [top]
"""
import collections
import csv
import re
import sys

sass_csv, dis, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 12
rows = list(csv.reader(open(sass_csv)))
h = rows[1]
cols = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
data = [r for r in rows[2:] if len(r) > max(cols)]
start = int(data[0][0], 16)
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
agg = collections.defaultdict(collections.Counter)
for r in data:
    ln = off2line.get(int(r[0], 16) - start)
    for i in cols:
        if r[i].isdigit():
            agg[ln][h[i]] += int(r[i])
tot = sum(sum(c.values()) for c in agg.values())
for ln, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(c.values())
    print(f"line {ln}: {100 * s / tot:5.1f}%  " + ", ".join(f"{k[6:]} {v}" for k, v in c.most_common(4)))
