"""Eager timing of the 8B-shaped decode SSM step (B=64), with and without group sums (the
harness of profiles/r02_decode_fusion.txt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import DeviceBlock, Dims  # noqa: E402

d = Dims("mamba2", 4096, 8192, 128, 128, 64, 8, 4)
B = 64
blk = DeviceBlock(synth.random_qblock(d, "W8A8", 5), "cuda")
zx = torch.randint(-100, 100, (B, d.in_proj_out), dtype=torch.int8, device="cuda")
h = torch.randint(-100, 100, (B, d.n_heads, d.head_dim, d.d_state), dtype=torch.int8, device="cuda")
c = torch.randint(-100, 100, (B, 3, d.conv_dim), dtype=torch.int8, device="cuda")
y = torch.zeros((B, d.d_inner), device="cuda")
ws = torch.zeros(ops.mamba2_decode_ws_bytes(blk.decode_params, B), dtype=torch.uint8, device="cuda")
for _ in range(3):
    ops.mamba2_decode_step_int8(blk.decode_params, B, zx, c, h, y=y, ws=ws)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20):
    ops.mamba2_decode_step_int8(blk.decode_params, B, zx, c, h, y=y, ws=ws)
e.record()
torch.cuda.synchronize()
print("decode step us", s.elapsed_time(e) / 20 * 1e3)
gs = torch.zeros((B, d.d_inner // 128), dtype=torch.int32, device="cuda")
for _ in range(3):
    ops.mamba2_decode_step_int8(blk.decode_params, B, zx, c, h, y=y, ws=ws, gsum=gs)
torch.cuda.synchronize()
s.record()
for _ in range(20):
    ops.mamba2_decode_step_int8(blk.decode_params, B, zx, c, h, y=y, ws=ws, gsum=gs)
e.record()
torch.cuda.synchronize()
print("three-launch decode step (+ group sums) us", s.elapsed_time(e) / 20 * 1e3)
