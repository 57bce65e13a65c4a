"""Launch one decode projection GEMM shape a few times (for ncu --set full captures).
usage: prof_gemm.py [in|out|head] [w4a8|w8a8]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "in"
kind = sys.argv[2] if len(sys.argv) > 2 else "w4a8"
M, N, K = {"in": (64, 18560, 4096), "out": (64, 4096, 8192), "head": (64, 256000, 4096)}[which]
dev = "cuda"
a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device=dev)
out = torch.empty((M, N), dtype=torch.float32, device=dev)
nb = 4
if kind == "w4a8":
    w = [torch.randint(0, 256, (ops.w4_bytes(N, K),), dtype=torch.uint8, device=dev) for _ in range(nb)]
    ws = [ops.tile_group_scales(torch.rand(N, K // 128, device=dev) * 1e-2) for _ in range(nb)]
    run = lambda i: ops.gemm_w4a8(a, w[i % nb], ws[i % nb], 128, 0.01, N, ops.EPI_F32, out)  # noqa: E731
else:
    w = [torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev) for _ in range(nb)]
    al = torch.rand(N, device=dev) * 1e-3
    run = lambda i: ops.gemm_w8a8(a, w[i % nb], al, ops.EPI_F32, out)  # noqa: E731
for i in range(6):
    run(i)
torch.cuda.synchronize()
print("ok")
