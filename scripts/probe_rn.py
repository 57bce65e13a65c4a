"""Per-CTA timeline of state_ring_norm_kernel (probe build -DSQ_RN_TRACE, probe/probe_rn.so), 8B shapes, B=64."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_22879_b200 import _lib, ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import DeviceBlock, Dims  # noqa: E402

lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "probe", "probe_rn.so"))
_lib._lib = lib
d = Dims("mamba2", 4096, 8192, 128, 128, 64, 8, 4)
B = 64
blk = DeviceBlock(synth.random_qblock(d, "W8A8", 5), "cuda")
zx = torch.randint(-100, 100, (B, d.in_proj_out), dtype=torch.int8, device="cuda")
h = torch.randint(-100, 100, (B, d.n_heads, d.head_dim, d.d_state), dtype=torch.int8, device="cuda")
c = torch.randint(-100, 100, (B, 3, d.conv_dim), dtype=torch.int8, device="cuda")
y = torch.zeros((B, d.d_inner), device="cuda")
ws = torch.zeros(ops.mamba2_decode_ws_bytes(blk.decode_params, B), dtype=torch.uint8, device="cuda")
for _ in range(4):
    ops.mamba2_decode_step_int8(blk.decode_params, B, zx, c, h, y=y, ws=ws)
    torch.cuda.synchronize()
buf = np.zeros((1024, 8), np.uint64)
lib.sq_probe_rn_trace(buf.ctypes.data_as(ctypes.c_void_p))
n = int((buf[:, 0] > 0).sum())
b = buf[:n].astype(np.int64)
t0 = b[:, 0].min()
for j, nm in [(0, "start"), (1, "cons loop end"), (2, "drain end"), (4, "counter end")]:
    v = (b[:, j] - t0) / 1e3
    print(f"{nm:14s} min {v.min():8.2f} med {np.median(v):8.2f} max {v.max():8.2f} argmax {v.argmax()}")
for j, nm in [(3, "norm us"), (5, "counter gpu-op us")]:
    v = b[:, j] / 1e3
    print(f"{nm:18s} min {v.min():8.2f} med {np.median(v):8.2f} max {v.max():8.2f} argmax {v.argmax()}")
print("norms per CTA max", b[:, 6].max(), "sum", b[:, 6].sum())
