"""Time the W4A8 GEMM probe variants built by scripts/probe_w4.sh (in_proj / out_proj / head shapes)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import _lib, ops  # noqa: E402

SHAPES = [("in_proj", 64, 18560, 4096), ("out_proj", 64, 4096, 8192), ("head", 64, 256000, 4096), ("in b1", 1, 18560, 4096)]
if os.environ.get("PROBE_LONGK"):   # steady state: one unit per SM, 4x the K of in_proj
    SHAPES = [("long K", 64, 18560, 8192), ("in_proj", 64, 18560, 4096)]
dev = "cuda"
for name in sys.argv[1:]:
    _lib._lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "probe", f"probe_{name}.so"))
    for sname, M, N, K in SHAPES:
        a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device=dev)
        out = torch.empty((M, N), dtype=torch.float32, device=dev)
        nb = max(1, min(6, int(2e9 // (N * K))))
        w4 = [torch.randint(0, 256, (ops.w4_bytes(N, K),), dtype=torch.uint8, device=dev) for _ in range(nb)]
        ws = [ops.tile_group_scales(torch.rand(N, K // 128, device=dev)) for _ in range(nb)]
        for i in range(3):
            ops.gemm_w4a8(a, w4[i % nb], ws[i % nb], 128, 0.01, N, ops.EPI_F32, out)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st), torch.cuda.graph(g, stream=st):
            for i in range(20):
                ops.gemm_w4a8(a, w4[i % nb], ws[i % nb], 128, 0.01, N, ops.EPI_F32, out)
        torch.cuda.current_stream().wait_stream(st)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 20
        print(f"{name:8s} {sname:9s} {t * 1e3:8.1f} us  {(N * K / 2 + N * K / 32) / t / 1e6:7.0f} GB/s", flush=True)
