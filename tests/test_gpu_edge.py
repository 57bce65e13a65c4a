"""Edge cases of the C-ABI ops on the GPU: empty batches are no-ops (outputs untouched, no
launch error), and bad shapes / layouts raise the reference's exception classes
(errors.py:4-25) instead of computing.  Oracle-free: these check boundary behaviour only."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ops():
    from paper_2503_22879_b200 import ops
    return ops


def test_empty_batches_are_noops(cuda):
    ops = _ops()
    dev = cuda
    # row kernels
    x = torch.empty((0, 512), device=dev)
    assert ops.rmsnorm_quant(x, torch.ones(512, device=dev), 1e-5, 0.1).shape == (0, 512)
    assert ops.rmsnorm_f32(x, torch.ones(512, device=dev), 1e-5).shape == (0, 512)
    assert ops.quantize_f32(x, 0.1).shape == (0, 512)
    assert ops.gate_norm_had_quant(torch.empty((0, 1024), device=dev), torch.ones(1024, device=dev), 1e-5,
                                   0.1).shape == (0, 1024)
    # GEMMs with M = 0
    a = torch.empty((0, 256), dtype=torch.int8, device=dev)
    w = torch.randint(-127, 128, (128, 256), dtype=torch.int8, device=dev)
    alpha = torch.ones(128, device=dev)
    assert ops.gemm_w8a8(a, w, alpha, ops.EPI_F32).shape == (0, 128)
    # conv with B = 0 or T = 0 leaves the cache untouched
    C = 64
    cache = torch.randint(-100, 100, (2, 3, C), dtype=torch.int8, device=dev)
    before = cache.clone()
    wt, bt = torch.randn((C, 4), device=dev), torch.zeros(C, device=dev)
    s = torch.full((C,), 0.02, device=dev)
    ops.conv1d_int8(torch.empty((0, C), dtype=torch.int8, device=dev), wt, bt, s, s, 2, 0, cache, True)
    assert torch.equal(cache, before)
    torch.cuda.synchronize()


def test_bad_shapes_and_layouts_raise(cuda):
    from paper_2503_22879_b200.errors import LayoutError, ShapeError
    ops = _ops()
    dev = cuda
    # CPU tensors: no CPU fallback
    with pytest.raises(LayoutError):
        ops.quantize_f32(torch.zeros((4, 16)), 0.1)
    # wrong dtype
    with pytest.raises((LayoutError, ShapeError)):
        ops.quantize_f32(torch.zeros((4, 16), dtype=torch.float16, device=dev), 0.1)
    # non-positive scale
    with pytest.raises((ShapeError, ValueError, RuntimeError)):
        ops.quantize_f32(torch.zeros((4, 16), device=dev), 0.0)
    # W4A16 GEMV: the group must divide K
    with pytest.raises((ShapeError, RuntimeError)):
        ops.gemv_w4a16(torch.zeros((1, 48), device=dev), torch.zeros(48, dtype=torch.uint8, device=dev),
                       torch.ones((2, 1), device=dev), 32, 2)
    # state / cache buffers smaller than the launch dimensions (would be out-of-bounds writes)
    C = 64
    wt, bt, sc = torch.randn((C, 4), device=dev), torch.zeros(C, device=dev), torch.full((C,), 0.02, device=dev)
    with pytest.raises(ShapeError):
        ops.conv1d_int8(torch.zeros((2 * 5, C), dtype=torch.int8, device=dev), wt, bt, sc, sc, 2, 5,
                        torch.zeros((1, 3, C), dtype=torch.int8, device=dev))
    with pytest.raises(ShapeError):
        ops.conv1d_update_int8(torch.zeros((3, C), dtype=torch.int8, device=dev), wt, bt, sc, sc,
                               torch.zeros((2, 3, C), dtype=torch.int8, device=dev))
    from paper_2503_22879_b200 import synth
    from paper_2503_22879_b200.ssm_block import DeviceBlock, Dims
    blk = DeviceBlock(synth.random_qblock(Dims("mamba2", 256, 512, 64, 8, 64, 2, 4), "W8A8", 1), dev)
    st = blk.new_state(2, dev)
    zx = torch.zeros((3, blk.dims.in_proj_out), dtype=torch.int8, device=dev)
    with pytest.raises(ShapeError):   # state and conv cache for 2 sequences, step for 3
        ops.mamba2_decode_step_int8(blk.decode_params, 3, zx, st.conv_cache, st.h)
    # conv kernel longer than supported
    with pytest.raises((ShapeError, RuntimeError)):
        ops.conv1d_int8(torch.zeros((4, 8), dtype=torch.int8, device=dev), torch.zeros((8, 9), device=dev),
                        torch.zeros(8, device=dev), torch.ones(8, device=dev), torch.ones(8, device=dev), 1, 4,
                        torch.zeros((1, 8, 8), dtype=torch.int8, device=dev))
    torch.cuda.synchronize()


def test_gemm_ragged_shapes_exact(cuda):
    """N not a multiple of the 128-row tile and M not a multiple of the token tile."""
    ops = _ops()
    r = np.random.default_rng(17)
    for M, N, K in ((1, 130, 128), (17, 257, 384), (65, 200, 256)):
        a = r.integers(-128, 128, (M, K)).astype(np.int8)
        w = r.integers(-127, 128, (N, K)).astype(np.int8)
        got = ops.gemm_w8a8(torch.as_tensor(a, device=cuda), torch.as_tensor(w, device=cuda),
                            torch.ones(N, device=cuda), ops.EPI_I32).cpu().numpy()
        assert np.array_equal(got, a.astype(np.int64) @ w.astype(np.int64).T)
