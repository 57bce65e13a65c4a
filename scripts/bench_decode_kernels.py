"""CUDA-event timing (warm, back-to-back) of the Mamba2-8B decode kernels at b=64."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import Dims  # noqa: E402


def timeit(fn, reps=20):
    """Per-call device time: `reps` calls captured in one CUDA graph (no host launch cost)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    for _ in range(2):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (5 * reps) * 1e3


d = Dims("mamba2", 4096, 8192, 128, 128, 64, 8, 4)
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = "cuda"
blk = synth.device_qblock(d, "W4A8", 0, dev)
st = blk.new_state(B, dev)
st.h.copy_(torch.randint(-100, 100, st.h.shape, dtype=torch.int8, device=dev))
zx = torch.randint(-128, 128, (B, d.in_proj_out), dtype=torch.int8, device=dev)
di, gn = d.d_inner, d.n_state_groups * d.d_state
y = torch.randn((B, di), device=dev)
yq = torch.empty((B, di), dtype=torch.int8, device=dev)
xbc = torch.empty(ops.mamba2_decode_ws_bytes(blk.decode_params, B), dtype=torch.uint8, device=dev)
u = torch.randint(-100, 100, (B, d.d_model), dtype=torch.int8, device=dev)
cv = torch.empty((B, d.conv_dim), dtype=torch.int8, device=dev)
state_bytes = st.h.numel() * 2
res = {}
sts = [st] + [blk.new_state(B, dev) for _ in range(2)]   # 3 x 67 MB > L2: every call streams from HBM
cnt = [0]


def step_rot():
    s_ = sts[cnt[0] % 3]
    cnt[0] += 1
    ops.mamba2_decode_step_int8(blk.decode_params, B, zx, s_.conv_cache, s_.h, yq, y, xbc)


res["decode_step (conv+state+norm)"] = timeit(step_rot, reps=21)
res["conv1d_update_int8 (old)"] = timeit(lambda: ops.conv1d_update_int8(zx[:, di:2 * di + 2 * gn], blk.conv_w, blk.conv_b,
                                                                         blk.conv_in_scale, blk.conv_out_scale,
                                                                         st.conv_cache, cv))
res["state_update_int8 (old)"] = timeit(lambda: ops.state_update_int8(blk.params, B, cv[:, :di], cv[:, di:di + gn],
                                                                       cv[:, di + gn:], zx[:, 2 * di + 2 * gn:], zx[:, :di],
                                                                       st.h, y))
res["gate_norm_had_quant (old)"] = timeit(lambda: ops.gate_norm_had_quant(y, blk.norm_w, 1e-5, blk.s_y, True, yq))
res["in_proj W4A8"] = timeit(lambda: blk.in_proj.a8(u, ops.EPI_QUANT, zx, blk.in_out_scale))
res["out_proj W4A8"] = timeit(lambda: blk.out_proj.a8(yq, ops.EPI_F32, None))
ugs = u.view(B, -1, 128).sum(-1, dtype=torch.int32)
ygs = yq.view(B, -1, 128).sum(-1, dtype=torch.int32)
res["in_proj W4A8 +gsum"] = timeit(lambda: blk.in_proj.a8(u, ops.EPI_QUANT, zx, blk.in_out_scale, ugs))
res["out_proj W4A8 +gsum"] = timeit(lambda: blk.out_proj.a8(yq, ops.EPI_F32, None, gsum=ygs))
tiny_x = torch.zeros((1, 16), device=dev)
tiny_q = torch.empty((1, 16), dtype=torch.int8, device=dev)
res["launch floor (1x16 quantize)"] = timeit(lambda: ops.quantize_f32(tiny_x, 0.1, tiny_q), reps=50)
h2 = torch.empty_like(st.h)
res["copy state 67MB (torch)"] = timeit(lambda: h2.copy_(st.h))
big_a = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
big_b = torch.empty(1 << 30, dtype=torch.uint8, device=dev)
res["copy 1GiB (torch)"] = timeit(lambda: big_b.copy_(big_a), reps=3)
print(f"copy 1GiB: {2 * (1 << 30) / res['copy 1GiB (torch)'] / 1e3:.0f} GB/s")
for k, v in res.items():
    extra = ""
    if "state" in k or "decode_step" in k:
        extra = f"  state r+w {state_bytes / v / 1e3:.0f} GB/s"
    print(f"{k:36s} {v:8.2f} us{extra}", flush=True)
