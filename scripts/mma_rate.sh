SQ_GEMM_DBG=64 timeout 120 python scripts/prof_kernels.py gemm 2>&1 | grep mma-rate | sort | uniq
SQ_GEMM_DBG=66 timeout 120 python scripts/prof_kernels.py gemm 2>&1 | grep "cta 0" | tail -8
SQ_GEMM_DBG=64 timeout 120 python - <<'PY' 2>&1 | grep mma-rate | sort | uniq
import torch
from paper_2503_22879_b200 import ops
for mode in (1, 2):
    ops.set_gemm_mode(mode)
    for M, N, K in ((64, 18560, 4096), (128, 18560, 4096), (16, 18560, 4096)):
        a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device="cuda")
        w4 = torch.randint(0, 256, (ops.w4_bytes(N, K),), dtype=torch.uint8, device="cuda")
        sg = torch.randint(1, 16, (N, K // 128), dtype=torch.int8, device="cuda")
        ops.gemm_w4a8(a, w4, sg, 128, torch.rand(N, device="cuda"), N, ops.EPI_F32)
    w8 = torch.randint(-127, 128, (N, K), dtype=torch.int8, device="cuda")
    ops.gemm_w8a8(a, w8, torch.rand(N, device="cuda"), ops.EPI_F32)
torch.cuda.synchronize()
PY
