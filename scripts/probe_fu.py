"""Per-CTA timeline of the fused decode step (probe build with -DSQ_FU_TRACE, probe/probe_fu.so)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_22879_b200 import _lib, ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import DeviceBlock, Dims  # noqa: E402

lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "probe", "probe_fu.so"))
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
buf = np.zeros((1024, 13), np.uint64)
lib.sq_probe_fu_trace(buf.ctypes.data_as(ctypes.c_void_p))
n = int((buf[:, 0] > 0).sum())
b = buf[:n].astype(np.int64)
t0 = b[:, 0].min()
rel = (b[:, :7] - t0) / 1e3
names = ["start", "producer", "x", "B|C", "counter", "cons loop", "drain"]
for j, nm in enumerate(names):
    v = rel[:, j]
    print(f"{nm:10s} min {v.min():8.2f} med {np.median(v):8.2f} max {v.max():8.2f}  argmax {v.argmax()}")
print("norms per CTA: max", b[:, 7].max(), "total", b[:, 7].sum(), "norm us mean", (b[:, 8].sum() / max(1, b[:, 7].sum())) / 1e3)
for j, nm in zip(range(9, 13), ["prod wait empty", "x wait empty", "B|C wait empty", "cons wait full"]):
    v = b[:, j] / 1e3
    print(f"{nm:16s} min {v.min():8.2f} med {np.median(v):8.2f} max {v.max():8.2f}")
worst = rel[:, 6].argmax()
print("worst CTA", worst, rel[worst], "norms", b[worst, 7], "norm us", b[worst, 8] / 1e3)
ev = np.zeros((64, 6), np.uint64)
lib.sq_probe_fu_events(ev.ctypes.data_as(ctypes.c_void_p))
e0 = ev[ev > 0].min()
r = np.where(ev > 0, (ev.astype(np.int64) - np.int64(e0)) / 1e3, np.nan)
print("CTA 0 tile events (us): prod issue | x arrive | B|C arrive | cons got full | w0 release | w15 release")
for i in range(min(40, 64)):
    print(f"{i:3d} " + " ".join(f"{v:8.2f}" for v in r[i]))
nt = np.zeros(8, np.uint64)
lib.sq_probe_fu_norm(nt.ctypes.data_as(ctypes.c_void_p))
print("CTA 0 norm phases (us from entry): loads+ss, reduce+scale, FWHT, quant:",
      " ".join(f"{(int(nt[k]) - int(nt[0])) / 1e3:.2f}" for k in range(1, 5)))
