"""Mamba1-2.8B b=1 decode, SSM half of a block: the one-launch kernel (sq_mamba1_decode_step_int8)
vs the five-launch chain, each replayed 20x from a CUDA graph (per-step device time), plus a
few bare launches for ncu captures.   python scripts/prof_m1dec.py [B]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import EPS_NORM, DeviceBlock, Dims  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
d = Dims("mamba1", 2560, 5120, 16, 1, 5120, 1, 4, dt_rank=160)
blk = DeviceBlock(synth.random_qblock(d, "W8A8", seed=7), "cuda")
di, R = d.d_inner, d.dt_rank
zx = torch.randint(-128, 128, (B, 2 * di), dtype=torch.int8, device="cuda")
h = torch.randint(-100, 100, (B, 1, di, 16), dtype=torch.int8, device="cuda")
cc = torch.randint(-100, 100, (B, 3, di), dtype=torch.int8, device="cuda")
ws = torch.zeros(ops.mamba1_decode_ws_bytes(blk.m1_decode_params, B), dtype=torch.uint8, device="cuda")
yq = torch.empty((B, di), dtype=torch.int8, device="cuda")
cv = torch.empty((B, di), dtype=torch.int8, device="cuda")
xd = torch.empty((B, R + 32), dtype=torch.int8, device="cuda")
dtq = torch.empty((B, di), dtype=torch.int8, device="cuda")
y = torch.empty((B, di), device="cuda")


def fused():
    ops.mamba1_decode_step_int8(blk.m1_decode_params, B, zx, cc, h, ws, yq)


def chain():
    ops.conv1d_update_int8(zx[:, di:], blk.conv_w, blk.conv_b, blk.conv_in_scale, blk.conv_out_scale, cc, cv)
    blk.x_proj.a8(cv, ops.EPI_QUANT, xd, blk.xproj_out_scale)
    blk.dt_proj.a8(xd[:, :R], ops.EPI_QUANT, dtq, blk.dt_scale)
    ops.selective_scan_int8(blk.params, B, 1, cv, dtq, xd[:, R:], zx[:, :di], h, True, y)
    ops.gate_norm_had_quant(y, blk.norm_w, EPS_NORM, blk.s_y, blk.hadamard, yq)


for name, fn in (("fused", fused), ("chain", chain)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s), torch.cuda.graph(g, stream=s):
        for _ in range(20):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:6s} B={B}: {e0.elapsed_time(e1) * 1000 / 20:.2f} us per step (graph of 20)", flush=True)

if os.environ.get("M1D_TRACE"):   # probe build with -DSQ_M1D_TRACE: phase timestamps of CTA 0 / last CTA
    from paper_2503_22879_b200 import _lib
    _lib._lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "probe", "probe_trace.so"))
    for _ in range(5):
        chain()
        fused()
    torch.cuda.synchronize()
    t = ws[64:64 + 160].view(torch.int64).cpu().tolist()
    names = ["start", "pdl_wait", "conv", "bar1", "x_proj", "bar2", "scan", "bar3", "norm"]
    for row, off in (("cta0", 0), ("last", 10)):
        print(row, " ".join(f"{n}={(t[off + k] - t[0]) / 1000:.2f}" for k, n in enumerate(names)))
