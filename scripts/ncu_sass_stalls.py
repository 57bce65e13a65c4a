"""Per-SASS-instruction stall breakdown from an ncu report (source page, sass view): the hottest
instructions with their dominant stall reasons, optionally restricted to an address window."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ri = [h.index(c) for c in reasons]
tot = {c: 0 for c in reasons}
for r in data:
    for c, i in zip(reasons, ri):
        if r[i].isdigit():
            tot[c] += int(r[i])
print("totals:", sorted(((v, k) for k, v in tot.items()), reverse=True)[:8])
top = sorted(data, key=lambda r: -int(r[si]) if r[si].isdigit() else 0)[:n]
for r in top:
    rs = sorted(((int(r[i]), c[6:]) for c, i in zip(reasons, ri) if r[i].isdigit() and int(r[i]) > 0), reverse=True)[:3]
    print(f"{r[si]:>5} {r[ie]:>8} {r[0][-5:]} {r[1][:56]:56s} {rs}")
