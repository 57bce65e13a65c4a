"""Time the Mamba1 int8 selective scan probe variants (probe/probe_<name>.so) at the 2.8B prefill
shape (B=1, T=1024, d_inner=5120, N=16)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import _lib, ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import DeviceBlock, Dims  # noqa: E402

d = Dims("mamba1", 2560, 5120, 16, 1, 5120, 1, 4, dt_rank=160)
blk = DeviceBlock(synth.random_qblock(d, "W8A8", 3), "cuda")
B, T = 1, 1024
g = torch.Generator(device="cuda")
g.manual_seed(0)
x = torch.randint(-100, 100, (B * T, 5120), dtype=torch.int8, device="cuda", generator=g)
dt = torch.randint(-100, 100, (B * T, 5120), dtype=torch.int8, device="cuda", generator=g)
bc = torch.randint(-100, 100, (B * T, 32), dtype=torch.int8, device="cuda", generator=g)
z = torch.randint(-100, 100, (B * T, 5120), dtype=torch.int8, device="cuda", generator=g)
ref = None
for name in sys.argv[1:]:
    _lib._lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "..", "probe", f"probe_{name}.so"))
    st = torch.zeros((B, 5120, 16), dtype=torch.int8, device="cuda")
    y = torch.empty((B * T, 5120), device="cuda")
    for _ in range(3):
        st.zero_()
        ops.selective_scan_int8(blk.params, B, T, x, dt, bc, z, st, False, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        ops.selective_scan_int8(blk.params, B, T, x, dt, bc, z, st, False, y)
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = y.clone()
    print(f"{name:8s} {e0.elapsed_time(e1) * 100:.1f} us  max|dy|/max|y| {((y - ref).abs().max() / ref.abs().max()).item():.2e}",
          flush=True)
