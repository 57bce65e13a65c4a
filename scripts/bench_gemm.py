"""Time the A8 GEMM modes on the decode/prefill projection shapes (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops  # noqa: E402

SHAPES = [("in_proj 8B b64", 64, 18560, 4096), ("out_proj 8B b64", 64, 4096, 8192),
          ("head 8B b64", 64, 256000, 4096), ("in_proj 8B b1", 1, 18560, 4096),
          ("in_proj 2.7B prefill", 16384, 10576, 2560), ("out_proj 2.7B prefill", 16384, 2560, 5120)]


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dev = "cuda"
for name, M, N, K in SHAPES:
    a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device=dev)
    alpha = torch.rand(N, device=dev) * 1e-3
    out = torch.empty((M, N), dtype=torch.float32, device=dev)
    w4 = torch.randint(0, 256, (ops.w4_bytes(N, K),), dtype=torch.uint8, device=dev)
    sg = torch.randint(1, 16, (N, K // 128), dtype=torch.int8, device=dev)
    w8 = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
    for mode in (0, 1, 2):
        ops.set_gemm_mode(mode)
        t4 = timeit(lambda: ops.gemm_w4a8(a, w4, sg, 128, alpha, N, ops.EPI_F32, out))
        t8 = timeit(lambda: ops.gemm_w8a8(a, w8, alpha, ops.EPI_F32, out)) if mode != 2 else float("nan")
        b4 = N * K / 2 + N * K / 128 + M * K + M * N * 4
        b8 = N * K + M * K + M * N * 4
        ops_ = 2.0 * M * N * K
        print(f"{name:24s} mode={mode} W4A8 {t4*1e3:8.1f} us {b4/t4/1e6:7.0f} GB/s {ops_/t4/1e9:7.1f} TOPS | "
              f"W8A8 {t8*1e3:8.1f} us {b8/t8/1e6:7.0f} GB/s {ops_/t8/1e9:7.1f} TOPS", flush=True)
ops.set_gemm_mode(1)
