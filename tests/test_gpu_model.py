"""GPU parity at model level (tiny configs) and at full Mamba2-8B layer shapes."""
import numpy as np
import pytest
import torch

from oracle import pipeline as opl
from oracle import qblock as oq
from oracle import ssm_block as osb

pytestmark = pytest.mark.gpu


def _tiny_model(profile, n_layers=2, variant="mamba2"):
    if variant == "mamba2":
        d = osb.Dims("mamba2", 256, 512, 64, 8, 64, 2, 4)
    else:
        d = osb.Dims("mamba1", 256, 512, 16, 1, 512, 1, 4, dt_rank=32)
    fm = opl.cmd_gen_toy(d, n_layers, seed=0)
    toks = opl.calib_tokens(512, 2, 64)
    return fm, toks, opl.cmd_quantize(fm, toks, profile)


@pytest.mark.parametrize("profile,variant", [("W8A8", "mamba2"), ("W4A8", "mamba2"), ("W4A16", "mamba2"),
                                             ("W8A8", "mamba1"), ("W4A16", "mamba1")])
def test_model_prefill_logits(cuda, profile, variant):
    from paper_2503_22879_b200.model import QuantizedMambaLM
    fm, toks, qm = _tiny_model(profile, variant=variant)
    ref, _ = opl.quant_forward(qm, toks[0, :40])
    lm = QuantizedMambaLM(qm, cuda)
    lg, _ = lm.prefill(torch.as_tensor(toks[:1, :40], device=cuda), all_logits=True)
    rel = np.abs(lg.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert rel < 1e-2, rel       # north_star: rel-err ≤ 1e-2 on logits


def test_model_batched_prefill_equals_per_sequence(cuda):
    from paper_2503_22879_b200.model import QuantizedMambaLM
    fm, toks, qm = _tiny_model("W8A8")
    lm = QuantizedMambaLM(qm, cuda)
    both, _ = lm.prefill(torch.as_tensor(toks[:, :32], device=cuda), all_logits=True)
    both = both.cpu().numpy().reshape(2, 32, -1)
    for i in range(2):
        one, _ = lm.prefill(torch.as_tensor(toks[i:i + 1, :32], device=cuda), all_logits=True)
        assert np.array_equal(one.cpu().numpy(), both[i]), "batch items are independent (SPEC.md:350)"


def test_generate_graph_equals_eager_and_oracle(cuda):
    from paper_2503_22879_b200.model import QuantizedMambaLM
    fm, toks, qm = _tiny_model("W8A8")
    lm = QuantizedMambaLM(qm, cuda)
    prompt = torch.as_tensor(toks[:2, :16], device=cuda)
    g = lm.generate(prompt, 12, use_graph=True).cpu().numpy()
    e = lm.generate(prompt, 12, use_graph=False).cpu().numpy()
    assert np.array_equal(g, e)
    ref = opl.generate(qm, toks[0, :16], 12)
    agree = (g[0] == ref).mean()
    assert agree >= 0.75, (g[0], ref)


def _to_oracle(pqb):
    od = osb.Dims(**vars(pqb.dims))
    return oq.QBlock(od, pqb.profile, oq.QLinear(**vars(pqb.in_proj)), oq.QLinear(**vars(pqb.out_proj)),
                     pqb.conv_weight, pqb.conv_bias, pqb.a_log, pqb.d_param, pqb.dt_bias, pqb.norm_weight,
                     pqb.head_group, s_u=pqb.s_u, in_out_scale=pqb.in_out_scale, conv_in_scale=pqb.conv_in_scale,
                     conv_out_scale=pqb.conv_out_scale, state_scale=pqb.state_scale, s_y=pqb.s_y)


def test_mamba2_8b_layer_decode_b64(cuda):
    """One Mamba2-8B-shaped W4A8 layer, decode b=64 from a random int8 state (C3 shapes)."""
    from paper_2503_22879_b200.ssm_block import DeviceBlock, SsmState
    from paper_2503_22879_b200 import synth
    d = osb.Dims("mamba2", 4096, 8192, 128, 128, 64, 8, 4)
    pqb = synth.random_qblock(d, "W4A8", seed=3)
    qb = _to_oracle(pqb)
    B = 64
    r = np.random.default_rng(0)
    u = (r.standard_normal((B, d.d_model))).astype(np.float32)
    h0 = r.integers(-100, 100, (B, d.n_heads, d.head_dim, d.d_state)).astype(np.int8)
    c0 = r.integers(-100, 100, (B, d.conv_dim, 3)).astype(np.int8)
    blk = DeviceBlock(pqb, cuda)
    st = SsmState(torch.as_tensor(h0, device=cuda), torch.as_tensor(np.ascontiguousarray(c0.transpose(0, 2, 1)),
                                                                     device=cuda))
    from paper_2503_22879_b200 import ops
    codes = ops.quantize_f32(torch.as_tensor(u, device=cuda), blk.s_u)
    out = blk.forward_codes(codes, B, 1, st, True).cpu().numpy()
    ro, rh, rc = oq.decode_step_batched(u, qb, h0, c0)
    rel = np.abs(out - ro).max() / np.abs(ro).max()
    assert rel < 2e-2, rel
    hd = np.abs(st.h.cpu().numpy().astype(np.int32) - rh.astype(np.int32))
    assert hd.max() <= 1 and (hd > 0).mean() < 1e-3
    assert np.array_equal(st.conv_cache.cpu().numpy().transpose(0, 2, 1), rc)
    for i in (0, 63):      # the batched oracle equals the per-sequence oracle
        ro1, rs1 = oq.block_forward_quantized(u[i:i + 1], qb, oq.QState(h0[i], c0[i]))
        assert np.array_equal(ro1[0], ro[i]) and np.array_equal(rs1.h, rh[i])


def test_product_quantize_pipeline_on_gpu(cuda):
    """The product's own host pipeline (gen-toy -> calibrate on the GPU -> quantize) feeding the
    GPU model: logits within 1e-2 of the oracle pipeline's quantized model."""
    from paper_2503_22879_b200 import cli
    from paper_2503_22879_b200.model import QuantizedMambaLM
    from paper_2503_22879_b200.ssm_block import Dims
    dims = ("mamba2", 256, 512, 64, 8, 64, 2, 4)
    fm = cli.cmd_gen_toy(Dims(*dims), 2, seed=0)
    toks = cli.calib_tokens(512, 2, 64)
    qm = cli.cmd_quantize(fm, toks, "W4A8", device="cuda")
    ofm = opl.cmd_gen_toy(osb.Dims(*dims), 2, seed=0)
    oqm = opl.cmd_quantize(ofm, toks, "W4A8")
    ref, _ = opl.quant_forward(oqm, toks[0, :32])
    lm = QuantizedMambaLM(qm, cuda)
    lg, _ = lm.prefill(torch.as_tensor(toks[:1, :32], device=cuda), all_logits=True)
    rel = np.abs(lg.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert rel < 1e-2, rel


def test_quant_archive_loads_into_gpu_model(cuda, tmp_path):
    """A quantized artifact (ModelArchive) read back into QuantizedMambaLM gives
    the same logits as the in-memory quantized model (u4 payloads repacked once on load)."""
    from paper_2503_22879_b200 import archive, cli
    from paper_2503_22879_b200.model import QuantizedMambaLM
    from paper_2503_22879_b200.ssm_block import Dims
    fm = cli.cmd_gen_toy(Dims("mamba2", 256, 512, 64, 8, 64, 2, 4), 2, seed=3)
    toks = cli.calib_tokens(512, 2, 32)
    qm = cli.cmd_quantize(fm, toks, ["W4A8", "W8A8"], device="cuda", emb_bits=4)
    p = str(tmp_path / "q.bin")
    archive.write_quant_model(qm, p)
    x = torch.as_tensor(toks[:1, :24], device=cuda)
    a, _ = QuantizedMambaLM(qm, cuda).prefill(x, all_logits=True)
    b, _ = QuantizedMambaLM(archive.read_quant_model(p), cuda).prefill(x, all_logits=True)
    assert torch.equal(a, b)


@pytest.mark.parametrize("profile", ["W8A8", "W4A8"])
def test_4bit_embedding_logits(cuda, profile):
    """Head-to-toe with 4-bit embedding rows: logits within 1e-2 of the oracle."""
    from paper_2503_22879_b200.model import QuantizedMambaLM
    d = osb.Dims("mamba2", 256, 512, 64, 8, 64, 2, 4)
    fm = opl.cmd_gen_toy(d, 2, seed=0)
    toks = opl.calib_tokens(512, 2, 64)
    qm = opl.cmd_quantize(fm, toks, profile, emb_bits=4)
    assert qm.emb_codes.min() >= -8 and qm.emb_codes.max() <= 7
    ref, _ = opl.quant_forward(qm, toks[0, :40])
    lm = QuantizedMambaLM(qm, cuda)
    assert lm.emb_bits == 4 and lm.emb_codes.dtype == torch.uint8
    lg, _ = lm.prefill(torch.as_tensor(toks[:1, :40], device=cuda), all_logits=True)
    rel = np.abs(lg.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert rel < 1e-2, rel


def _tp_worker(rank, world, port, q, profile):
    """One rank of the head-shard model: its blocks are head shards, the out_proj partials are
    all-reduced over the group (gloo here: both ranks share cuda:0; NCCL on a multi-GPU box)."""
    import os
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import dataclasses
    import numpy as np
    import torch
    from oracle import pipeline as opl
    from oracle import qblock as oq
    from oracle import ssm_block as osb
    from paper_2503_22879_b200 import cli, parallel
    from paper_2503_22879_b200 import dist as pdist
    from paper_2503_22879_b200.model import QuantizedMambaLM
    from paper_2503_22879_b200.ssm_block import Dims
    pdist.init("gloo")
    try:
        dev = torch.device("cuda", 0)
        d = Dims("mamba2", 256, 512, 64, 8, 64, 2, 4, norm_groups=world)   # shard-local recipe
        fm = cli.cmd_gen_toy(d, 2, seed=31)
        toks = cli.calib_tokens(512, 2, 32)
        qm = cli.cmd_quantize(fm, toks, profile, device="cuda")
        shard = dataclasses.replace(qm, dims=parallel.shard_qblock(qm.blocks[0], world, rank).dims,
                                    blocks=[parallel.shard_qblock(b, world, rank) for b in qm.blocks])
        lm = QuantizedMambaLM(shard, dev, tp_group=torch.distributed.group.WORLD)
        prompt = np.asarray(toks[0, :12])
        gl, gst = lm.prefill(torch.as_tensor(prompt[None], device=dev))
        nxt = int(torch.argmax(gl[0]).item())
        gl2 = lm.decode_step(torch.tensor([nxt], dtype=torch.int32, device=dev), gst)
        if rank == 0:   # the unsharded oracle model of the same recipe
            ql = lambda x: None if x is None else oq.QLinear(x.kind, x.codes, x.s_ch, x.s_group, x.group)  # noqa: E731
            ob = [oq.QBlock(osb.Dims(**vars(b.dims)), b.profile, ql(b.in_proj), ql(b.out_proj), b.conv_weight,
                            b.conv_bias, b.a_log, b.d_param, b.dt_bias, b.norm_weight, b.head_group, s_u=b.s_u,
                            in_out_scale=b.in_out_scale, conv_in_scale=b.conv_in_scale,
                            conv_out_scale=b.conv_out_scale, state_scale=b.state_scale, s_y=b.s_y,
                            hadamard=b.hadamard) for b in qm.blocks]
            om = opl.QuantModel(osb.Dims(**vars(qm.dims)), qm.profiles, np.asarray(qm.emb_codes),
                                np.asarray(qm.emb_scale), [np.asarray(w) for w in qm.layer_norms], ob,
                                np.asarray(qm.final_norm), ql(qm.head), np.float32(qm.s_head))
            rl, rst = opl.quant_forward(om, prompt)
            rl2, _ = opl.quant_forward(om, [nxt], rst)
            rel = lambda a, b: float(np.abs(a - b).max() / np.abs(b).max())   # noqa: E731
            q.put((rel(gl.cpu().numpy()[0], rl[-1]), rel(gl2.cpu().numpy()[0], rl2[-1])))
        pdist.barrier(world)
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.parametrize("profile", ["W8A8", "W4A8"])
def test_head_shard_model_world2(cuda, profile):
    """QuantizedMambaLM in head-shard mode (tp_group): 2 ranks (gloo, one GPU) each run their
    heads of every block and all-reduce the out_proj partials; prefill and a decode step give the
    unsharded oracle model's logits (rel <= 1e-2, north_star)."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tp_worker, args=(r, 2, port, q, profile)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    r1, r2 = q.get(timeout=5)
    assert r1 <= 1e-2 and r2 <= 1e-2, (r1, r2)


@pytest.mark.gpu
def test_gptq_on_gpu_projection_shape(cuda):
    """GPTQ on the GPU at a projection shape (1024 x 2560, group 128, 512
    calibration rows): lower proxy loss than round-to-nearest, codes in range, same result as the
    float64-Hessian CPU run up to float32 sweep rounding (codes differ in < 1e-3 of entries)."""
    import numpy as np
    from paper_2503_22879_b200 import quantizer
    r = np.random.default_rng(7)
    w = (r.standard_normal((1024, 2560)) / 50).astype(np.float32)
    X = (r.standard_normal((512, 2560)) * np.exp(r.uniform(-1, 1, 2560))).astype(np.float32)
    g = quantizer.gptq_quantize_weight(w, X, 4, 128, device=cuda)
    rt = quantizer.quantize_weight_w4(w, 128)
    deq = lambda q: (q.payload.to(torch.float64).cpu() * q.layout.expand(q.shape).to(torch.float64).cpu()).numpy()
    loss = lambda wq: float(np.square(X.astype(np.float64) @ (w.astype(np.float64) - wq).T).sum())
    assert loss(deq(g)) < loss(deq(rt))
    c = g.payload.cpu().numpy()
    assert c.min() >= -8 and c.max() <= 7
    gc = quantizer.gptq_quantize_weight(w[:64], X, 4, 128, device="cpu")
    assert (gc.payload.numpy() != c[:64]).mean() < 1e-3
