"""A/B parity of two decode-step paths on identical inputs: sq_mamba2_decode_step_int8 without and
with the group-sum output (the harness used for the fused-kernel experiments of
profiles/r02_decode_fusion.txt; those kernels are in commits 6df4bab and 3e7018f)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import DeviceBlock, Dims  # noqa: E402

for dims, B in [(("mamba2", 256, 512, 64, 8, 64, 2, 4), 3), (("mamba2", 4096, 8192, 128, 128, 64, 8, 4), 64)]:
    d = Dims(*dims)
    blk = DeviceBlock(synth.random_qblock(d, "W8A8", 5), "cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(1)
    zx = torch.randint(-100, 100, (B, d.in_proj_out), dtype=torch.int8, device="cuda", generator=g)
    h0 = torch.randint(-100, 100, (B, d.n_heads, d.head_dim, d.d_state), dtype=torch.int8, device="cuda", generator=g)
    c0 = torch.randint(-100, 100, (B, 3, d.conv_dim), dtype=torch.int8, device="cuda", generator=g)
    res = []
    for fused in (True, False):
        h, c = h0.clone(), c0.clone()
        y = torch.zeros((B, d.d_inner), device="cuda")
        gs = None if fused else torch.zeros((B, d.d_inner // 128), dtype=torch.int32, device="cuda")
        yq = ops.mamba2_decode_step_int8(blk.decode_params, B, zx, c, h, y=y, gsum=gs)
        torch.cuda.synchronize()
        res.append((h, c, y, yq))
    (h1, c1, y1, q1), (h2, c2, y2, q2) = res
    print(dims[2], "state max diff", (h1.int() - h2.int()).abs().max().item(), "frac", ((h1 != h2).float().mean().item()))
    print("   conv equal", torch.equal(c1, c2), "x part", torch.equal(c1[:, :, :d.d_inner], c2[:, :, :d.d_inner]))
    print("   y rel", ((y1 - y2).abs().max() / y2.abs().max()).item())
    print("   yq max diff", (q1.int() - q2.int()).abs().max().item(), "frac", (q1 != q2).float().mean().item())
