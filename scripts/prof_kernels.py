"""Launch the decode hot kernels a few times each (for ncu --set full captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import Dims  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
d = Dims("mamba2", 4096, 8192, 128, 128, 64, 8, 4)
B = 64
dev = "cuda"
blk = synth.device_qblock(d, "W4A8", 0, dev)
st = blk.new_state(B, dev)
st.h.copy_(torch.randint(-100, 100, st.h.shape, dtype=torch.int8, device=dev))
u = torch.randint(-100, 100, (B, d.d_model), dtype=torch.int8, device=dev)
zx = blk.in_proj.a8(u, ops.EPI_QUANT, None, blk.in_out_scale)
di, gn = d.d_inner, d.n_state_groups * d.d_state
cv = ops.conv1d_update_int8(zx[:, di:2 * di + 2 * gn], blk.conv_w, blk.conv_b, blk.conv_in_scale, blk.conv_out_scale,
                            st.conv_cache)
y = torch.empty((B, di), device=dev)
for _ in range(3):
    if which in ("all", "fused"):
        cc = st.conv_cache
        ops.mamba2_decode_step_int8(blk.decode_params, B, zx, cc, st.h, y=y)
    if which in ("all", "state"):
        ops.state_update_int8(blk.params, B, cv[:, :di], cv[:, di:di + gn], cv[:, di + gn:], zx[:, 2 * di + 2 * gn:],
                              zx[:, :di], st.h, y)
    if which in ("all", "gemm"):
        blk.in_proj.a8(u, ops.EPI_QUANT, zx, blk.in_out_scale)
    if which in ("all", "gemm", "gemm_out"):
        yq8 = torch.randint(-100, 100, (B, d.d_inner), dtype=torch.int8, device=dev)
        blk.out_proj.a8(yq8, ops.EPI_F32, None)
    if which in ("all", "norm"):
        yq = ops.gate_norm_had_quant(y, blk.norm_w, 1e-5, blk.s_y, True)
        ops.rmsnorm_quant(torch.randn(B, d.d_model, device=dev), torch.ones(d.d_model, device=dev), 1e-5, 0.03)
torch.cuda.synchronize()
print("ok")
