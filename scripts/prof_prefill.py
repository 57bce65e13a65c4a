"""Launch the prefill non-GEMM kernels (conv, chunked SSD, gated norm) at the prefill27b
shapes a few times each, for ncu --set full captures and quick per-kernel timing.

    python scripts/prof_prefill.py [conv|ssd|norm|all] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import Dims  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
d = Dims("mamba2", 2560, 5120, 128, 80, 64, 1, 4)
B, T = 8, 2048
M = B * T
dev = "cuda"
blk = synth.device_qblock(d, "W8A8", 0, dev)
di, gn = d.d_inner, d.n_state_groups * d.d_state
g = torch.Generator(device=dev)
g.manual_seed(3)
zx = torch.randint(-100, 100, (M, 2 * di + 2 * gn + d.n_heads), generator=g, dtype=torch.int8, device=dev)
xbc = zx[:, di:2 * di + 2 * gn]
cache = torch.zeros((B, d.conv_kernel - 1, di + 2 * gn), dtype=torch.int8, device=dev)
cv = torch.empty((M, di + 2 * gn), dtype=torch.int8, device=dev)
state = torch.zeros((B, d.n_heads, d.head_dim, d.d_state), dtype=torch.int8, device=dev)
y = torch.empty((M, di), device=dev)
ev = {k: (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for k in ("conv", "ssd", "norm")}
tm = {k: [] for k in ev}
for r in range(reps):
    if which in ("all", "conv"):
        ev["conv"][0].record()
        ops.conv1d_int8(xbc, blk.conv_w, blk.conv_b, blk.conv_in_scale, blk.conv_out_scale, B, T, cache, False, cv)
        ev["conv"][1].record()
    if which in ("all", "ssd"):
        ev["ssd"][0].record()
        ops.ssd_scan_int8(blk.params, B, T, cv[:, :di], cv[:, di:di + gn], cv[:, di + gn:], zx[:, 2 * di + 2 * gn:],
                          zx[:, :di], state, False, y)
        ev["ssd"][1].record()
    if which in ("all", "norm"):
        ev["norm"][0].record()
        yq = ops.gate_norm_had_quant(y, blk.norm_w, 1e-5, blk.s_y, True)
        ev["norm"][1].record()
    torch.cuda.synchronize()
    for k in ev:
        if which in ("all", k):
            tm[k].append(ev[k][0].elapsed_time(ev[k][1]) * 1e3)
for k, v in tm.items():
    if v:
        print(f"{k}: last {v[-1]:.1f} us  min {min(v):.1f} us")
if which in ("gemm",):
    u = torch.randint(-100, 100, (M, d.d_model), generator=g, dtype=torch.int8, device=dev)
    yq = torch.randint(-100, 100, (M, di), generator=g, dtype=torch.int8, device=dev)
    h = torch.zeros((M, d.d_model), device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for r_ in range(reps):
        e0.record()
        blk.in_proj.a8(u, ops.EPI_QUANT, zx, blk.in_out_scale)
        e1.record()
        torch.cuda.synchronize()
        t_in = e0.elapsed_time(e1) * 1e3
        e0.record()
        blk.out_proj.a8(yq, ops.EPI_RESID, h)
        e1.record()
        torch.cuda.synchronize()
        print(f"in_proj {t_in:.1f} us  out_proj {e0.elapsed_time(e1) * 1e3:.1f} us")
