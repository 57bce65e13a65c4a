import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_22879_b200 import ops
M, N, K = (int(v) for v in sys.argv[1:4])
a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device="cuda")
alpha = torch.rand(N, device="cuda") * 1e-3
out = torch.empty((M, N), dtype=torch.float32, device="cuda")
w4 = torch.randint(0, 256, (ops.w4_bytes(N, K),), dtype=torch.uint8, device="cuda")
sg = torch.randint(1, 16, (N, K // 128), dtype=torch.int8, device="cuda")
for _ in range(3):
    ops.gemm_w4a8(a, w4, sg, 128, alpha, N, ops.EPI_F32, out)
torch.cuda.synchronize()
