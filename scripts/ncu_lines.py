"""Per-source-line instruction count and stall samples for one kernel of an ncu report.

    python scripts/ncu_lines.py <sass.csv> <nvdisasm -g -c dump> <mangled-name-substring> [topN]
"""
import collections
import csv
import re
import sys

sass_csv, dis, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
rows = list(csv.reader(open(sass_csv)))
# the export may hold several kernels: take the section whose "Kernel Name" row mentions fn
secs, cur_sec = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur_sec = [r]
        secs.append(cur_sec)
    elif cur_sec is not None:
        cur_sec.append(r)
sec = next((x for x in secs if fn in x[0][1] or fn.split("_")[-1] in x[0][1]), secs[0])
h = sec[1]
data = [r for r in sec[2:] if len(r) > 5 and r[0].startswith("0x")]
ie, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
start = int(data[0][0], 16)
val = {int(r[0], 16) - start: (int(r[ie]) if r[ie].isdigit() else 0, int(r[si]) if r[si].isdigit() else 0)
       for r in data}
inside, cur, off2 = False, None, {}
for l in open(dis).read().splitlines():
    if l.startswith(".text.") and fn in l:
        inside = True
        continue
    if inside and l.startswith(".text."):
        break
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r'\s+/\*([0-9a-f]{4,})\*/', l)
    if m:
        off2[int(m.group(1), 16)] = cur
ai, ast = collections.Counter(), collections.Counter()
for o, (n, s) in val.items():
    ai[off2.get(o)] += n
    ast[off2.get(o)] += s
ti, ts = max(1, sum(ai.values())), max(1, sum(ast.values()))
print(f"warp-instr {ti}  stall samples {ts}")
srcs = {}
for k, n in ast.most_common(top):
    txt = ""
    if k:
        if k[0] not in srcs:
            try:
                srcs[k[0]] = open(k[0]).read().splitlines()
            except OSError:
                srcs[k[0]] = []
        L = srcs[k[0]]
        txt = L[k[1] - 1].strip()[:70] if k[1] - 1 < len(L) else ""
    name = f"{k[0].split('/')[-1]}:{k[1]}" if k else "?"
    print(f"stall {100 * n / ts:5.1f}%  inst {100 * ai[k] / ti:5.1f}%  {name:22s} {txt}")
