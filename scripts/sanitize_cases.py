"""Small-shape invocations of every mbarrier / TMA / TMEM kernel, one launch each, for
compute-sanitizer (scripts/sanitize.sh): W4A8 GEMM (persistent and split-K cluster), W8A8 GEMM
(single and split-K), the fused decode step (prep + state ring + norm), both chunked-SSD engines,
the int8 conv and the gated norm, the W4A16 bf16 GEMV (mma.sync and row fallback) and the Mamba1
int8 scan (single pass and the time-chunked two-pass form) and the one-launch Mamba1 decode step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2503_22879_b200 import ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import DeviceBlock, Dims, block_forward_quantized  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = "cuda"
g = torch.Generator(device=dev)
g.manual_seed(0)


def run(name, fn):
    if which in ("all", name):
        fn()
        torch.cuda.synchronize()
        print("ok", name, flush=True)


def w4a8():
    for M, N, K in ((64, 512, 1024), (16, 256, 8192), (64, 2048, 512)):   # persistent / split-K / multi-unit
        a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device=dev, generator=g)
        w = torch.randint(0, 256, (ops.w4_bytes(N, K),), dtype=torch.uint8, device=dev, generator=g)
        ws = ops.tile_group_scales(torch.rand(N, K // 128, device=dev, generator=g))
        ops.gemm_w4a8(a, w, ws, 128, 0.01, N, ops.EPI_F32)


def w8a8():
    for M, N, K in ((64, 512, 1024), (16, 256, 8192), (300, 256, 512)):
        a = torch.randint(-128, 128, (M, K), dtype=torch.int8, device=dev, generator=g)
        w = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev, generator=g)
        ops.gemm_w8a8(a, w, torch.rand(N, device=dev, generator=g) * 1e-3, ops.EPI_F32)


def decode():
    d = Dims("mamba2", 256, 512, 128, 8, 64, 2, 4)
    blk = DeviceBlock(synth.random_qblock(d, "W8A8", 1), dev)
    st = blk.new_state(3, dev)
    zx = torch.randint(-100, 100, (3, d.in_proj_out), dtype=torch.int8, device=dev, generator=g)
    ops.mamba2_decode_step_int8(blk.decode_params, 3, zx, st.conv_cache, st.h)


def ssd():
    d = Dims("mamba2", 256, 1024, 128, 16, 64, 2, 4)
    blk = DeviceBlock(synth.random_qblock(d, "W8A8", 2), dev)
    u = torch.randn(2 * 200, d.d_model, device=dev, generator=g)
    block_forward_quantized(u, blk, batch=2)       # conv, mma.sync SSD engine, gated norm, GEMMs
    T = 130
    xq = torch.randint(-100, 100, (T, 1024), dtype=torch.int8, device=dev, generator=g)
    bc = torch.randint(-100, 100, (T, 256), dtype=torch.int8, device=dev, generator=g)
    dt = torch.randint(-100, 100, (T, 16), dtype=torch.int8, device=dev, generator=g)
    h = torch.zeros((1, 16, 64, 128), dtype=torch.int8, device=dev)
    y = torch.empty((T, 1024), device=dev)
    ops.ssd_scan_int8(blk.params, 1, T, xq, bc, bc, dt, xq, h, False, y, chunk=128)   # tcgen05 engine


def w4a16():
    from paper_2503_22879_b200.ssm_block import pack_u4_host
    for M, N, K, group in ((1, 100, 256, 128), (5, 64, 512, 64), (3, 40, 160, 32)):
        codes = np.random.default_rng(0).integers(-8, 8, (N, K)).astype(np.int8)
        w = ops.repack_w4a16(torch.as_tensor(pack_u4_host(codes), device=dev), N, K, group)
        x = torch.randn(M, K, device=dev, generator=g)
        ops.gemv_w4a16(x, w, torch.rand(N, K // group, device=dev, generator=g), group, N)


def m1():
    d = Dims("mamba1", 64, 64, 16, 1, 64, 1, 4, dt_rank=8)
    blk = DeviceBlock(synth.random_qblock(d, "W8A8", 3), dev)
    for T in (48, 700):   # single pass / time-chunked
        x, dt, z = (torch.randint(-100, 100, (T, 64), dtype=torch.int8, device=dev, generator=g) for _ in range(3))
        bc = torch.randint(-100, 100, (T, 32), dtype=torch.int8, device=dev, generator=g)
        st = torch.zeros((1, 64, 16), dtype=torch.int8, device=dev)
        ops.selective_scan_int8(blk.params, 1, T, x, dt, bc, z, st, False, torch.empty((T, 64), device=dev))
    # one-launch decode step (grid barriers), twice on one workspace (self-resetting counters)
    B = 2
    zx = torch.randint(-100, 100, (B, 128), dtype=torch.int8, device=dev, generator=g)
    st = torch.zeros((B, 1, 64, 16), dtype=torch.int8, device=dev)
    cc = torch.zeros((B, 3, 64), dtype=torch.int8, device=dev)
    ws = torch.zeros(ops.mamba1_decode_ws_bytes(blk.m1_decode_params, B), dtype=torch.uint8, device=dev)
    for _ in range(2):
        ops.mamba1_decode_step_int8(blk.m1_decode_params, B, zx, cc, st, ws)


run("w4a8", w4a8)
run("w8a8", w8a8)
run("decode", decode)
run("ssd", ssd)
run("w4a16", w4a16)
run("m1", m1)
