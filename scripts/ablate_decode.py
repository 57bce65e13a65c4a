"""In-graph ablation of the Mamba2-8B W4A8 b=64 decode step (profiling only).

Captures the decode CUDA graph with one class of launches removed at a time and reports the
step time, so each kernel class's marginal in-graph cost (PDL overlap included) is
step(all) - step(without it).  Outputs are garbage in the ablated graphs; only time matters.

    python scripts/ablate_decode.py [--layers 56]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from paper_2503_22879_b200 import ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import Dims  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=56)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
d = Dims("mamba2", 4096, 8192, 128, 128, 64, 8, 4)
lm = synth.synthetic_lm(d, a.layers, "W4A8", 256000, "cuda")
states = lm.new_states(a.batch)

orig_gemm, orig_norm = ops.gemm_w4a8, ops.rmsnorm_quant


def timed(label, skip_in=False, skip_out=False, skip_head=False, skip_rms=False, stages=7):
    def gemm(a_, w4, sg, group, alpha, N, epi=ops.EPI_F32, out=None, col_scale=None, gsum=None):
        is_head = N > 20000
        is_out = epi == ops.EPI_RESID
        if (is_head and skip_head) or (is_out and skip_out) or (not is_head and not is_out and skip_in):
            return out
        return orig_gemm(a_, w4, sg, group, alpha, N, epi, out, col_scale, gsum)

    def norm(x, gamma, eps, s, out=None, gsum=None):
        if skip_rms:
            return out
        return orig_norm(x, gamma, eps, s, out, gsum)

    ops.gemm_w4a8, ops.rmsnorm_quant = gemm, norm
    ops.set_decode_stages(stages)
    try:
        g, tok, lg, ws = lm.capture_decode(a.batch, states)
    finally:
        ops.gemm_w4a8, ops.rmsnorm_quant = orig_gemm, orig_norm
        ops.set_decode_stages(7)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    print(f"{label:34s} {ms * 1e3:9.1f} us/step  {ms * 1e3 / a.layers:7.2f} us/layer", flush=True)
    del g
    return ms


full = timed("all")
timed("no in_proj", skip_in=True)
timed("no out_proj", skip_out=True)
timed("no head", skip_head=True)
timed("no rmsnorm", skip_rms=True)
timed("no prep (stages 6)", stages=6)
timed("no ring (stages 5)", stages=5)
timed("no norm_had (stages 3)", stages=3)
timed("only ring (stages 2, no gemm/rms)", skip_in=True, skip_out=True, skip_head=True, skip_rms=True, stages=2)
timed("only gemms", stages=0, skip_rms=True)
