"""W8A8 at M=1 (the Mamba1-2.8B decode projections) through sq_gemm_w8a8, 20 launches in a CUDA
graph over rotating weights (weights from HBM).  A dp4a GEMV was measured against the tcgen05
path with this script and lost on every shape but x_proj."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops  # noqa: E402

M = int(os.environ.get("GEMV_M", "1"))
for name, N, K in (("in_proj", 10240, 2560), ("out_proj", 2560, 5120), ("x_proj", 192, 5120), ("dt_proj", 5120, 160)):
    a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device="cuda")
    nb = max(2, min(8, int(4e8 // (N * K))))
    w = [torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda") for _ in range(nb)]
    al = torch.rand(N, device="cuda") * 1e-3
    out = torch.empty(M, N, device="cuda")
    for i in range(3):
        ops.gemm_w8a8(a, w[i % nb], al, ops.EPI_F32, out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
        for i in range(20):
            ops.gemm_w8a8(a, w[i % nb], al, ops.EPI_F32, out)
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 50
    print(f"{name} M={M}: {us:.1f} us  {N * K / us / 1e3:.0f} GB/s", flush=True)
