"""Per-kernel table of an ncu launch-list CSV: python scripts/launch_table.py gpurun_out/x.csv"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) > vi:
        v = float(r[vi].replace(",", ""))
        v = v / 1000 if r[ui] in ("nsecond", "ns") else v * 1000 if r[ui] in ("msecond", "ms") else v
        agg[r[ki][:80]][0] += 1
        agg[r[ki][:80]][1] += v
tot = sum(t for _, t in agg.values())
print(f"# {sum(n for n, _ in agg.values())} launches, sum {tot / 1000:.3f} ms")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:10.1f} us {100 * t / tot:5.1f}% {n:5d} {t / n:8.2f}  {k}")
