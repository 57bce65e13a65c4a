"""In-graph timing of the decode W4A8 projections in TS (A from TMEM) vs SS (A in smem) mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import Dims  # noqa: E402


def timeit(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * reps) * 1e3


d = Dims("mamba2", 4096, 8192, 128, 128, 64, 8, 4)
B = 64
dev = "cuda"
blks = [synth.device_qblock(d, "W4A8", i, dev) for i in range(3)]
u = torch.randint(-100, 100, (B, d.d_model), dtype=torch.int8, device=dev)
zx = torch.empty((B, d.in_proj_out), dtype=torch.int8, device=dev)
ugs = u.view(B, -1, 128).sum(-1, dtype=torch.int32)
cnt = [0]


def inp():
    b = blks[cnt[0] % 3]
    cnt[0] += 1
    b.in_proj.a8(u, ops.EPI_QUANT, zx, b.in_out_scale, ugs)


for mode in (1, 2):
    ops.set_gemm_mode(mode)
    print(f"mode {mode} ({'TS' if mode == 1 else 'SS'}): in_proj {timeit(inp):.2f} us")
