"""Time the A8 projection GEMMs on the decode / prefill shapes (CUDA events, distinct weight
buffers per launch so every launch streams its weights from HBM, as in the decode step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops  # noqa: E402

SHAPES = [("in_proj 8B b64", 64, 18560, 4096), ("out_proj 8B b64", 64, 4096, 8192),
          ("head 8B b64", 64, 256000, 4096), ("in_proj 8B b1", 1, 18560, 4096),
          ("in_proj 2.7B prefill", 16384, 10576, 2560), ("out_proj 2.7B prefill", 16384, 2560, 5120)]


def timeit(fn, reps=20):
    """Device time per launch of `reps` back-to-back launches replayed from a CUDA graph (no host
    launch overhead between them, like the decode step)."""
    for i in range(3):
        fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(reps):
                fn(i)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dev = "cuda"
for name, M, N, K in SHAPES:
    a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device=dev)
    alpha = torch.rand(N, device=dev) * 1e-3
    out = torch.empty((M, N), dtype=torch.float32, device=dev)
    nbuf = max(1, min(8, int(2e9 // (N * K))))     # rotate weights so they do not sit in L2
    w4 = [torch.randint(0, 256, (ops.w4_bytes(N, K),), dtype=torch.uint8, device=dev) for _ in range(nbuf)]
    ws = [ops.tile_group_scales(torch.rand(N, K // 128, device=dev) * 1e-2 + 1e-3) for _ in range(nbuf)]
    w8 = [torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev) for _ in range(nbuf)]
    t4 = timeit(lambda i: ops.gemm_w4a8(a, w4[i % nbuf], ws[i % nbuf], 128, 0.01, N, ops.EPI_F32, out))
    t8 = timeit(lambda i: ops.gemm_w8a8(a, w8[i % nbuf], alpha, ops.EPI_F32, out))
    b4 = N * K / 2 + N * K / 128 * 4 + M * K + M * N * 4
    b8 = N * K + M * K + M * N * 4
    ops_ = 2.0 * M * N * K
    print(f"{name:24s} W4A8 {t4*1e3:8.1f} us {b4/t4/1e6:7.0f} GB/s {ops_/t4/1e9:7.1f} TOPS (splits "
          f"{ops.gemm_w4a8_splits(M, N, K)}) | W8A8 {t8*1e3:8.1f} us {b8/t8/1e6:7.0f} GB/s {ops_/t8/1e9:7.1f} TOPS",
          flush=True)
