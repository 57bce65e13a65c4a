"""W4A16 GEMV at the Mamba2-8B decode shapes (b=1): in_proj 4096->18560, out_proj 8192->4096,
head 4096->256000.  CUDA-graph timing over rotating weight copies (weights from HBM); run under
ncu -k regex:gemv for a kernel capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops  # noqa: E402

M = int(os.environ.get("GEMV_M", "1"))
for name, N, K in (("in_proj", 18560, 4096), ("out_proj", 4096, 8192)):
    x = torch.randn(M, K, device="cuda")
    nb = 6
    w4 = [torch.randint(0, 256, (ops.w4a16_bytes(N, K, 128),), dtype=torch.uint8, device="cuda") for _ in range(nb)]
    sg = [torch.rand(N, K // 128, device="cuda") for _ in range(nb)]
    out = torch.empty(M, N, device="cuda")
    for i in range(3):
        ops.gemv_w4a16(x, w4[i % nb], sg[i % nb], 128, N, out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
        for i in range(20):
            ops.gemv_w4a16(x, w4[i % nb], sg[i % nb], 128, N, out)
    torch.cuda.current_stream().wait_stream(st)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 50
    print(f"{name} M={M}: {us:.1f} us  {(N * K / 2 + N * K / 128 * 4) / us / 1e3:.0f} GB/s", flush=True)
