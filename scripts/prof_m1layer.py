"""Mamba1-2.8B b=1 decode layer: the one-launch layer kernel (sq_mamba1_decode_layer_int8) vs the
four-launch chain (rmsnorm_quant + in_proj GEMM + one-launch SSM half + out_proj GEMM), each
replayed 20x from a CUDA graph; M1D_TRACE=1 with probe/probe_trace.so prints phase timestamps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import EPS_NORM, Dims  # noqa: E402

if os.environ.get("M1D_TRACE"):
    from paper_2503_22879_b200 import _lib
    _lib._lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "probe", "probe_trace.so"))
d = Dims("mamba1", 2560, 5120, 16, 1, 5120, 1, 4, dt_rank=160)
m = synth.synthetic_lm(d, 1, "W8A8", 512, "cuda", seed=4, head_kind="w8")
blk = m.blocks[0]
B = 1
h = torch.randn((B, d.d_model), device="cuda")
st = blk.new_state(B)
ws = m._workspace(B)
lp = m._m1_layer(0, blk)


def layer():
    ops.mamba1_decode_layer_int8(blk.m1_decode_params, lp, B, h, st.conv_cache, st.h, ws["m1ws"])


def chain():
    ops.rmsnorm_quant(h, m.layer_norms[0], EPS_NORM, blk.s_u, ws["u"])
    blk.forward_codes(ws["u"], B, 1, st, True, resid=h, ws=ws)


for name, fn in (("layer", layer), ("chain", chain)):
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
    print(f"{name}: {e0.elapsed_time(e1) * 1000 / 20:.2f} us per layer (graph of 20)", flush=True)
if os.environ.get("M1D_TRACE"):
    for _ in range(3):
        chain()
        layer()
    torch.cuda.synchronize()
    t = ws["m1ws"][64:64 + 160].view(torch.int64).cpu().tolist()
    names = ["start", "pdl_wait", "conv", "bar1", "x_proj", "bar2", "scan", "bar3", "end", "in_proj"]
    for row, off in (("cta0", 0), ("last", 10)):
        print(row, " ".join(f"{n}={(t[off + k] - t[0]) / 1000:.2f}" for k, n in enumerate(names)))
