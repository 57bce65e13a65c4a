"""W4A16 GEMV at the Mamba2-8B decode shapes (b=1): in_proj 4096->18560, out_proj 8192->4096.
Prints CUDA-event times; run under ncu -k regex:gemv for the kernel capture."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops  # noqa: E402

for name, N, K in (("in_proj", 18560, 4096), ("out_proj", 4096, 8192)):
    x = torch.randn(1, K, device="cuda")
    w4 = torch.randint(0, 256, (ops.w4_bytes(N, K),), dtype=torch.uint8, device="cuda")
    sg = torch.rand(N, K // 128, device="cuda")
    out = torch.empty(1, N, device="cuda")
    fn = lambda: ops.gemv_w4a16(x, w4, sg, 128, N, out)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 50
    print(f"{name}: {us:.1f} us  {(N * K / 2 + N * K / 128 * 4) / us / 1e3:.0f} GB/s", flush=True)
