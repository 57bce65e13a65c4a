"""Time W4A16 GEMV probe variants (probe/probe_<name>.so built by scripts/probe_build.sh gemv_w4a16.cu ...)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import _lib, ops  # noqa: E402

for name in sys.argv[1:]:
    _lib._lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "probe", f"probe_{name}.so"))
    for sname, N, K in (("in_proj", 18560, 4096), ("out_proj", 4096, 8192)):
        x = torch.randn(1, K, device="cuda")
        nb = 6
        w4 = [torch.randint(0, 256, (ops.w4a16_bytes(N, K, 128),), dtype=torch.uint8, device="cuda") for _ in range(nb)]
        sg = [torch.rand(N, K // 128, device="cuda") for _ in range(nb)]
        out = torch.empty(1, N, device="cuda")
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
        print(f"{name:10s} {sname}: {us:.1f} us  {(N * K / 2 + N * K / 128 * 4) / us / 1e3:.0f} GB/s", flush=True)
