"""Stall samples / instructions per gemm_a8_tc.cu source line (inline call sites resolved)
for the first kernel of an ncu source-page CSV export.

    python scripts/ncu_gemm_lines.py <sass.csv> <nvdisasm -gi -c dump> [topN]
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = [r]
        secs.append(cur)
    elif cur is not None:
        cur.append(r)
sec = secs[0]
print(sec[0][1][:100])
h = sec[1]
data = [r for r in sec[2:] if len(r) > 5 and r[0].startswith("0x")]
ie, si = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
start = int(data[0][0], 16)
val = {int(r[0], 16) - start: (int(r[ie]) if r[ie].isdigit() else 0, int(r[si]) if r[si].isdigit() else 0)
       for r in data}
tpl = re.search(r"gemm_tc_kernel<(.*?)>\(", sec[0][1]).group(1)
mang = "_ZN2sq14gemm_tc_kernelI" + "".join("Li%sE" % v for v in re.findall(r"\(int\)(\d+)", tpl)) + "EEv"
inside, cur, off2 = False, None, {}
for l in open(sys.argv[2]):
    if l.startswith(".text.") and mang in l:
        inside = True
        continue
    if inside and l.startswith(".text."):
        break
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?', l)
    if m:
        if m.group(3) and "gemm_a8_tc" in m.group(3):
            cur = int(m.group(4))
        elif "gemm_a8_tc" in m.group(1):
            cur = int(m.group(2))
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m:
        off2[int(m.group(1), 16)] = cur
ai, ast = collections.Counter(), collections.Counter()
for o, (n, s) in val.items():
    ai[off2.get(o)] += n
    ast[off2.get(o)] += s
ti, ts = max(1, sum(ai.values())), max(1, sum(ast.values()))
src = open("paper_2503_22879_b200/csrc/gemm_a8_tc.cu").read().splitlines()
print("instr", ti, "samples", ts)
for k, s in ast.most_common(top):
    txt = src[k - 1].strip()[:78] if k else ""
    print(f"stall {100 * s / ts:5.1f}% inst {100 * ai[k] / ti:5.1f}% line {k} {txt}")
