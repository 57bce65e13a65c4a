"""Summarise a gpurun_out/ pass into profiles/<tag>_*.txt (committed evidence).

    python scripts/summarize_profiles.py r01 [report_dir]
Reads gpurun_out/launches.csv (ncu --metrics gpu__time_duration.sum launch list of the
bench's timed steps) and every gpurun_out/*.ncu-rep (ncu --set full captures).
"""
import collections
import csv
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")


def launches(tag, src="launches.csv", name="launches"):
    p = os.path.join(OUT, src)
    if not os.path.exists(p):
        return
    rows = list(csv.reader(open(p)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h, data = rows[hi], rows[hi + 1:]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        k = r[ki].split("(")[0][:70]
        agg[k][0] += 1
        agg[k][1] += v
        tot += v
    lines = [f"# ncu launch list ({src}): gpu__time_duration.sum per launch, cold-cache + serialised",
             f"# {sum(a[0] for a in agg.values())} launches, sum {tot / 1e3:.3f} ms", "",
             f"{'total_us':>10} {'share':>6} {'n':>5} {'avg_us':>8}  kernel"]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{t:10.1f} {100 * t / tot:5.1f}% {n:5d} {t / n:8.2f}  {k}")
    open(os.path.join(PROF, f"{tag}_{name}.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Occupancy", "L2 Hit Rate", "Grid Size", "Block Size",
        "Executed Instructions", "Warp Cycles Per Issued Instruction", "One or More Eligible", "SM Frequency",
        "Dynamic Shared Memory Per Block"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg", "sm__cycles_elapsed.avg"]


def ncu_reports(tag, src=OUT):
    for rep in sorted(glob.glob(os.path.join(src, "*.ncu-rep"))):
        base = os.path.basename(rep)[:-8]
        det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(det.splitlines()))
        if not rows:
            continue
        h = rows[0]
        out = [f"# ncu --set full summary of {base}.ncu-rep"]
        cur = None
        for r in rows[1:]:
            d = dict(zip(h, r))
            if d.get("ID") != cur:
                cur = d.get("ID")
                out.append(f"\n## ID {cur}: {d.get('Kernel Name', '')[:150]}")
            if d.get("Metric Name") in WANT:
                out.append(f"  {d['Metric Name']:<40} {d['Metric Value']} {d['Metric Unit']}")
        rr = list(csv.reader(raw.splitlines()))
        if len(rr) > 2:
            hh, uu = rr[0], rr[1]
            for i, row in enumerate(rr[2:]):
                vals = [f"{n}={row[j]} {uu[j]}" for j, n in enumerate(hh) if n in RAW]
                out.append(f"\n## raw ID {i}: " + "; ".join(vals))
        open(os.path.join(PROF, f"{tag}_{base}.txt"), "w").write("\n".join(out) + "\n")
        print(f"wrote profiles/{tag}_{base}.txt")


if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(PROF, exist_ok=True)
    if len(sys.argv) > 2:   # only the ncu reports of one directory (e.g. gpurun_out/prof)
        ncu_reports(tag, sys.argv[2])
        sys.exit(0)
    launches(tag)
    launches(tag, "launches_prefill.csv", "launches_prefill")
    ncu_reports(tag)
    for src, dst in (("bench.json", "bench.json"), ("bench_ref.json", "bench_ref.json"),
                     ("bench_prefill.json", "bench_prefill.json"), ("pytest_gpu.log", "pytest_gpu.txt"),
                     ("bdk.log", "decode_kernels.txt"), ("stages.log", "decode_stages.txt"),
                     ("prefill_kernels.txt", "prefill_kernels.txt"), ("smoke.log", "smoke.txt"),
                     ("bench_other.json", "bench_other.json")):
        p = os.path.join(OUT, src)
        if os.path.exists(p):
            open(os.path.join(PROF, f"{tag}_{dst}"), "w").write(open(p).read())
            print(f"copied profiles/{tag}_{dst}")
