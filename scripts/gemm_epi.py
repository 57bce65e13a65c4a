"""Prefill out_proj (2.7B: 16384 x 2560 x 5120, W8A8) time per epilogue kind (profiling)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops  # noqa: E402

M, N, K = 16384, 2560, 5120
a = torch.randint(-100, 100, (M, K), dtype=torch.int8, device="cuda")
w8 = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
alpha = torch.rand(N, device="cuda") * 1e-4
out = torch.zeros((M, N), device="cuda")
out8 = torch.zeros((M, N), dtype=torch.int8, device="cuda")
cs = torch.full((N,), 0.05, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn in (("RESID", lambda: ops.gemm_w8a8(a, w8, alpha, ops.EPI_RESID, out)),
                 ("F32", lambda: ops.gemm_w8a8(a, w8, alpha, ops.EPI_F32, out)),
                 ("QUANT", lambda: ops.gemm_w8a8(a, w8, alpha, ops.EPI_QUANT, out8, cs))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"out_proj {name}: {e0.elapsed_time(e1) * 100:.1f} us", flush=True)
