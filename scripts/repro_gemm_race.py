"""Repeat a W4A8 GEMM and report where results deviate from the first run (race hunting)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_22879_b200 import ops  # noqa: E402
from paper_2503_22879_b200.ssm_block import pack_u4_host  # noqa: E402

M, N, K, group = (int(v) for v in (sys.argv[1:5] if len(sys.argv) > 4 else (300, 640, 1024, 128)))
epi = int(sys.argv[5]) if len(sys.argv) > 5 else ops.EPI_I32
r = np.random.default_rng(2)
a = r.integers(-128, 128, (M, K)).astype(np.int8)
codes = r.integers(-8, 8, (N, K)).astype(np.int8)
sg = r.integers(1, 16, (N, K // group)).astype(np.int8)
alpha = r.uniform(1e-4, 1e-2, N).astype(np.float32)
w8 = codes.astype(np.int64) * np.repeat(sg.astype(np.int64), group, axis=1)
ref = a.astype(np.int64) @ w8.T
tw = ops.repack_w4(torch.as_tensor(pack_u4_host(codes), device="cuda"), N, K)
ta, tsg, tal = (torch.as_tensor(x, device="cuda") for x in (a, sg, alpha))
ops.set_gemm_mode(int(os.environ.get("MODE", "1")))
yref = (ref.astype(np.float32) * alpha[None]).astype(np.float32)
bad = 0
for it in range(int(os.environ.get("REPS", "50"))):
    if epi == ops.EPI_I32:
        got = ops.gemm_w4a8(ta, tw, tsg, group, tal, N, ops.EPI_I32).cpu().numpy().astype(np.int64)
        d = got != ref
    else:
        got = ops.gemm_w4a8(ta, tw, tsg, group, tal, N, ops.EPI_F32).cpu().numpy()
        d = got != yref
        ref_ = yref
    if d.any():
        bad += 1
        rows, cols = np.nonzero(d)
        print(f"iter {it}: {d.sum()} wrong; tokens {np.unique(rows)[:12]} ({len(np.unique(rows))}), "
              f"cols {np.unique(cols // 128)} tiles, col range {cols.min()}-{cols.max()}; "
              f"sample got {got[rows[0], cols[0]]} want {(ref if epi == ops.EPI_I32 else yref)[rows[0], cols[0]]}")
print("bad runs", bad)
