"""Batch-shard data parallelism on CPU (gloo, world_size 2): every sequence is owned by exactly
one rank, max-over-ranks timing, and a sharded batched decode step (oracle arithmetic) gathered
in rank order equals the unsharded step bit for bit (sequences are independent)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2503_22879_b200 import dist as pdist


def test_shard_range_partitions():
    for n in (0, 1, 5, 64, 67):
        for world in (1, 2, 3, 8):
            rs = [pdist.shard_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        pdist.shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from oracle import qblock as oq
    from oracle import pipeline as opl
    from oracle import ssm_block as osb
    w, r, _ = pdist.init("gloo")
    try:
        assert (w, r) == (world, rank)
        mx = pdist.max_over_ranks(1.5 + rank, world)
        # tiny Mamba2 W8A8 block, 5 sequences, one decode step from random int8 states
        d = osb.Dims("mamba2", 256, 512, 64, 8, 64, 2, 4)
        fm = opl.cmd_gen_toy(d, 1, seed=0)
        toks = opl.calib_tokens(512, 2, 32)
        qb = opl.cmd_quantize(fm, toks, "W8A8").blocks[0]
        g = np.random.default_rng(5)
        nb = 5
        u = g.standard_normal((nb, d.d_model)).astype(np.float32)
        h = g.integers(-100, 100, (nb, d.n_heads, d.head_dim, d.d_state)).astype(np.int8)
        c = g.integers(-100, 100, (nb, d.conv_dim, d.conv_kernel - 1)).astype(np.int8)
        a, b = pdist.shard_range(nb, world, rank)
        out, hn, cn = oq.decode_step_batched(u[a:b], qb, h[a:b], c[a:b])
        counts = [e - s for s, e in (pdist.shard_range(nb, world, k) for k in range(world))]
        allo = pdist.gather_rows(torch.as_tensor(np.ascontiguousarray(out)), world, counts).numpy()
        allh = pdist.gather_rows(torch.as_tensor(np.ascontiguousarray(hn)), world, counts).numpy()
        if rank == 0:
            ref, href, _ = oq.decode_step_batched(u, qb, h, c)
            q.put((mx, bool(np.array_equal(allo, ref)), bool(np.array_equal(allh, href))))
        pdist.barrier(world)
    finally:
        torch.distributed.destroy_process_group()


def test_gloo_batch_shard_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    mx, same_out, same_h = q.get(timeout=5)
    assert mx == 2.5
    assert same_out and same_h


def _to_oracle_qb(pqb):
    from oracle import qblock as oq
    from oracle import ssm_block as osb
    ql = lambda q: None if q is None else oq.QLinear(q.kind, q.codes, q.s_ch, q.s_group, q.group)   # noqa: E731
    return oq.QBlock(osb.Dims(**vars(pqb.dims)), pqb.profile, ql(pqb.in_proj), ql(pqb.out_proj), pqb.conv_weight,
                     pqb.conv_bias, pqb.a_log, pqb.d_param, pqb.dt_bias, pqb.norm_weight, pqb.head_group,
                     s_u=pqb.s_u, in_out_scale=pqb.in_out_scale, conv_in_scale=pqb.conv_in_scale,
                     conv_out_scale=pqb.conv_out_scale, state_scale=pqb.state_scale, s_y=pqb.s_y,
                     hadamard=pqb.hadamard)


def _head_worker(rank, world, port, q, profile):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    from oracle import qblock as oq
    from paper_2503_22879_b200 import cli, parallel
    from paper_2503_22879_b200.ssm_block import Dims
    pdist.init("gloo")
    try:
        # head-shard recipe: grouped norm over d_inner / world channels, shard-local Hadamard
        d = Dims("mamba2", 256, 512, 64, 8, 64, 2, 4, norm_groups=world)
        fm = cli.cmd_gen_toy(d, 1, seed=2)
        qb = cli.cmd_quantize(fm, cli.calib_tokens(512, 2, 32), profile, device="cpu").blocks[0]
        u = np.random.default_rng(6).standard_normal((24, d.d_model)).astype(np.float32)
        part, st = oq.block_forward_quantized(u, _to_oracle_qb(parallel.shard_qblock(qb, world, rank)))
        t = torch.as_tensor(np.ascontiguousarray(part))
        torch.distributed.all_reduce(t)                   # the block's only collective
        hs = pdist.gather_rows(torch.as_tensor(st.h), world, [d.n_heads // world] * world).numpy()
        if rank == 0:
            ref, rst = oq.block_forward_quantized(u, _to_oracle_qb(qb))
            rel = float(np.abs(t.numpy() - ref).max() / np.abs(ref).max())
            q.put((rel, bool(np.array_equal(hs, rst.h))))
        pdist.barrier(world)
    finally:
        torch.distributed.destroy_process_group()


@pytest.mark.parametrize("profile", ["W8A8", "W4A8"])
def test_gloo_head_shard_world2(profile):
    """Head-shard mode: each rank runs its heads' shard of the block (in_proj rows,
    state groups, conv channels, grouped norm, shard-local Hadamard, out_proj K-slice) and one
    all-reduce of the out_proj partials reproduces the unsharded block: output within f32
    reassociation (rel 1e-5) and identical int8 state codes."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_head_worker, args=(r, 2, port, q, profile)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    rel, same_h = q.get(timeout=5)
    assert rel <= 1e-5, rel
    assert same_h
