"""Summarise an ncu report: SM active spread and the hottest source lines (stall samples)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
for i, k in enumerate(r[0]):
    if k in ("gpu__time_duration.sum", "sm__cycles_active.avg", "sm__cycles_active.max", "sm__cycles_active.min",
             "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread"):
        print(k, r[1][i], r[2][i])
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg, ex = collections.Counter(), collections.Counter()
hdr, cur, fname = None, None, None
for row in csv.reader(io.StringIO(src)):
    if row and row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row and row[0] == "Line No":
        hdr = row
        continue
    if len(row) >= 4 and row[0]:
        cur = (fname, int(row[0]), row[1][:90])
    if hdr and len(row) > 4 and row[2].startswith("0x"):
        try:
            agg[cur] += int(row[hdr.index("Warp Stall Sampling (All Samples)", 3)])
            ex[cur] += int(row[hdr.index("Instructions Executed", 3)])
        except ValueError:
            pass
print("total samples", sum(agg.values()))
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(v, ex[k], k)
