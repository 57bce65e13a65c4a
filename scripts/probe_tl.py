"""CTA-0 pipeline timeline of the W4A8 GEMM (probe build with -DSQ_W4_PROBE_TIMELINE):
rows = entry/exit and, per step of two groups: MMA committed, MMA got A stage, MMA got accumulator,
converter published, MMAs issued, MMA thread start-of-wait, MMA got activation stage (us from entry)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_22879_b200 import _lib, ops  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "tl"
lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "probe", f"probe_{name}.so"))
_lib._lib = lib
dev = "cuda"
for sname, M, N, K in [("in_proj", 64, 18560, 4096), ("out_proj", 64, 4096, 8192)]:
    a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device=dev)
    out = torch.empty((M, N), dtype=torch.float32, device=dev)
    w4 = [torch.randint(0, 256, (ops.w4_bytes(N, K),), dtype=torch.uint8, device=dev) for _ in range(3)]
    ws = [ops.tile_group_scales(torch.rand(N, K // 128, device=dev)) for _ in range(3)]
    for i in range(3):
        ops.gemm_w4a8(a, w4[i], ws[i], 128, 0.01, N, ops.EPI_F32, out)
        torch.cuda.synchronize()
    buf = np.zeros((12, 80), np.uint64)
    lib.sq_probe_w4_timeline(buf.ctypes.data_as(ctypes.c_void_p))
    t0 = buf[0, 0]
    rel = (buf.astype(np.int64) - np.int64(t0)) / 1e3
    names = ["entry/exit", "mma committed", "conv got w0", "conv converted", "conv pub", "mma issued", "mma wait0",
             "mma got act", "stream issue", "conv loaded", "conv tempty"]
    print(f"== {sname}: exit at {rel[0, 1]:.2f} us; promotion done {rel[0, 2]:.2f}, split-K: partial staged "
          f"{rel[0, 3]:.2f}, pre-sync {rel[0, 4]:.2f}, synced {rel[0, 5]:.2f}, reduced {rel[0, 6]:.2f}")
    G = (K // 128 if sname == "in_proj" else K // 128 // ops.gemm_w4a8_splits(M, N, K)) // 2   # steps
    for r in range(1, 11):
        vals = rel[r, :G]
        print(f"{names[r]:12s}", " ".join(f"{v:6.2f}" for v in vals))
