"""Quantized Mamba language model on the GPU: forward (prefill) and generate (decode).

Model wrapper (LEDGER G8): pre-norm residual stack
    h = E[tok];  for l: h += block_l(rmsnorm(h, ln_l));  logits = head(rmsnorm(h, ln_f))
Head-to-toe quantisation: embedding per-row int8 or 4-bit (u4packed rows,
PAPER.md:315-316), head W4A8 (or W8A8)
with a per-tensor 8-bit activation scale.  Every op is a kernel of
libssmquant_sm100.so; the residual stream stays fp32 in HBM.

Decode is one token per sequence per step; the whole step (embed →
56 blocks → head → argmax) is captured once in a CUDA graph and replayed, so the
host issues one launch per step and the argmax output feeds the next step on device.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .ssm_block import EPS_NORM, DeviceBlock, DeviceLinear, Dims, SsmState


@dataclass
class HostModel:
    """Host (numpy) quantized model: the product of `cli_pipeline.cmd_quantize`."""
    dims: Dims
    profiles: list
    emb_codes: np.ndarray
    emb_scale: np.ndarray
    layer_norms: list
    blocks: list
    final_norm: np.ndarray
    head: object
    s_head: float


class QuantizedMambaLM:
    """``tp_group`` (a torch.distributed group, head-shard mode, parallel.py): the blocks are this
    rank's head shards (shard-local norm / Hadamard recipe); each block's out_proj partial is
    summed over the group by one all_reduce (NCCL over NVLink on GPUs) before it joins the
    residual stream.  Embedding, pre-norms and the head are replicated."""

    def __init__(self, hm, device="cuda", tp_group=None):
        self.tp_group = tp_group
        self.tp_world = torch.distributed.get_world_size(tp_group) if tp_group is not None else 1
        self.dims = hm.dims
        self.device = torch.device(device)
        dev = self.device
        def t(a, dt):
            if isinstance(a, torch.Tensor):
                return a.to(device=dev, dtype=dt)
            return torch.as_tensor(np.asarray(a)).to(device=dev, dtype=dt)
        f = lambda a: t(a, torch.float32)
        extra = getattr(hm, "extra", None) or {}
        self.emb_bits = int(extra.get("emb_bits", 8))
        if self.emb_bits == 4:   # u4packed rows, half the bytes of the int8 table
            from .ssm_block import pack_u4_host
            codes = hm.emb_codes.cpu().numpy() if isinstance(hm.emb_codes, torch.Tensor) else np.asarray(hm.emb_codes)
            self.emb_codes = torch.as_tensor(pack_u4_host(codes), device=dev)
        else:
            self.emb_codes = t(hm.emb_codes, torch.int8)
        self.emb_scale = f(hm.emb_scale)
        self.layer_norms = [f(w) for w in hm.layer_norms]
        self.blocks = [b if isinstance(b, DeviceBlock) else DeviceBlock(b, dev) for b in hm.blocks]
        self.final_norm = f(hm.final_norm)
        self.s_head = np.float32(hm.s_head)
        self.head = hm.head if isinstance(hm.head, DeviceLinear) else DeviceLinear(hm.head, dev, self.s_head)
        self.vocab = self.head.N
        self._graphs = {}
        # Mamba1 W8A8 decode, one launch per whole layer (sq_mamba1_decode_layer_int8): bit-exact with
        # the 4-launch chain but not faster on B200 (32.0 vs 31.8 us per 2.8B layer with L2-warm
        # weights, 417 vs 454 tok/s in the bench with weights from HBM), so off
        self.fuse_layers = False

    @property
    def n_layers(self):
        return len(self.blocks)

    def weight_bytes(self):
        n = sum(b.weight_bytes for b in self.blocks) + self.head.nbytes
        return n

    # ------------------------------------------------------------------ state
    def new_states(self, batch: int):
        return [b.new_state(batch, self.device) for b in self.blocks]

    def _workspace(self, M: int):
        d = self.dims
        dev = self.device
        e = lambda shape, dt: torch.empty(shape, dtype=dt, device=dev)
        ws = {"h": e((M, d.d_model), torch.float32), "u": e((M, d.d_model), torch.int8),
              "zx": e((M, d.in_proj_out), torch.int8), "conv": e((M, d.conv_dim), torch.int8),
              "y": e((M, d.d_inner), torch.float32), "yq": e((M, d.d_inner), torch.int8),
              "hq": e((M, d.d_model), torch.int8), "logits": e((M, self.vocab), torch.float32),
              "tok": e((M,), torch.int32)}
        fused = [b for b in self.blocks if getattr(b, "fused_decode", False)]
        if fused:
            # zero-filled once: the fused decode kernel's counters live here (self-resetting)
            ws["dws"] = torch.zeros((ops.mamba2_decode_ws_bytes(fused[0].decode_params, M),), dtype=torch.uint8,
                                    device=dev)
        m1f = [b for b in self.blocks if getattr(b, "m1_fused_decode", False)]
        if m1f and M <= 8:
            # zero-filled once: the one-launch Mamba1 decode keeps its grid-barrier counters here
            ws["m1ws"] = torch.zeros((ops.mamba1_decode_ws_bytes(m1f[0].m1_decode_params, M),), dtype=torch.uint8,
                                     device=dev)
        if any(not b.a8 for b in self.blocks):
            ws.update(uf=e((M, d.d_model), torch.float32), zxf=e((M, d.in_proj_out), torch.float32),
                      convf=e((M, d.conv_dim), torch.float32), r=e((M, d.d_inner), torch.float32))
        if d.variant == "mamba1":
            ws.update(xd=e((M, d.dt_rank + 2 * d.d_state), torch.int8), dtq=e((M, d.d_inner), torch.int8))
        if self.tp_world > 1:
            ws["out"] = e((M, d.d_model), torch.float32)   # a block's out_proj partial before the all_reduce
        return ws

    # ------------------------------------------------------------------ forward
    def _m1_layer(self, l, blk):
        """Layer parameters of the one-launch Mamba1 decode layer (W8 in/out projections and the
        one-launch SSM half), built once per block; None when the block does not qualify."""
        if not self.fuse_layers or not getattr(blk, "m1_fused_decode", False):
            return None
        if blk.in_proj.kind != "w8" or blk.out_proj.kind != "w8":
            return None
        lp = getattr(blk, "_m1_layer_params", None)
        if lp is None:
            lp = ops.mamba1_layer_params(self.layer_norms[l], EPS_NORM, blk.s_u, self.dims.d_model, blk.in_proj.w,
                                         blk.in_proj.alpha, blk.in_out_scale, blk.out_proj.w, blk.out_proj.alpha)
            blk._m1_layer_params = lp
        return lp

    def _run(self, tok, B, T, states, state_in, ws, all_logits):
        """tok int32 [B*T] (b-major) → logits; every launch on the current stream."""
        h = ws["h"]
        if self.emb_bits == 4:
            ops.embed_u4(self.emb_codes, self.emb_scale, tok, self.dims.d_model, h)
        else:
            ops.embed_int8(self.emb_codes, self.emb_scale, tok, h)
        for l, blk in enumerate(self.blocks):
            st = states[l]
            lp = self._m1_layer(l, blk) if (T == 1 and state_in and self.tp_world == 1 and "m1ws" in ws) else None
            if lp is not None:   # Mamba1 W8A8 decode: the whole layer in one launch (decode_m1.cu)
                ops.mamba1_decode_layer_int8(blk.m1_decode_params, lp, B, h, st.conv_cache, st.h, ws["m1ws"])
                continue
            if blk.a8 and self.tp_world > 1:   # head shard: partial -> all_reduce -> residual
                ops.rmsnorm_quant(h, self.layer_norms[l], EPS_NORM, blk.s_u, ws["u"])
                part = blk.forward_codes(ws["u"], B, T, st, state_in, ws=ws)
                torch.distributed.all_reduce(part, op=torch.distributed.ReduceOp.SUM, group=self.tp_group)
                h.add_(part)
            elif blk.a8:
                ops.rmsnorm_quant(h, self.layer_norms[l], EPS_NORM, blk.s_u, ws["u"])
                blk.forward_codes(ws["u"], B, T, st, state_in, resid=h, ws=ws)
            else:
                # the pre-norm runs inside the in_proj GEMV (h is read before out_proj adds to it)
                blk.forward_a16(h, B, T, st, state_in, resid=h, ws=ws, u_norm=self.layer_norms[l])
        if all_logits:
            hs = h
            hq, lg = ws["hq"], ws["logits"]
        else:   # last token of every sequence only
            hs = h.view(B, T, -1)[:, T - 1, :]
            hq, lg = ws["hq"][:B], ws["logits"][:B]
        ops.rmsnorm_quant(hs, self.final_norm, EPS_NORM, self.s_head, hq)
        self.head.a8(hq, ops.EPI_F32, lg)
        return lg

    def prefill(self, tokens: torch.Tensor, states=None, all_logits=False):
        """tokens int [B×T] (CUDA) → (logits, states).  Fresh states unless given."""
        B, T = tokens.shape
        state_in = states is not None
        states = states if state_in else self.new_states(B)
        ws = self._workspace(B * T)
        tok = tokens.reshape(-1).to(torch.int32).contiguous()
        lg = self._run(tok, B, T, states, state_in, ws, all_logits)
        return lg.clone(), states

    def decode_step(self, tok: torch.Tensor, states, ws=None):
        """One decode step: tok int32 [B] → logits [B×V]; states updated in place."""
        B = tok.shape[0]
        ws = ws if ws is not None else self._workspace(B)
        return self._run(tok, B, 1, states, True, ws, True)

    # ------------------------------------------------------------------ graphs
    def capture_decode(self, batch: int, states):
        """Capture embed→blocks→head→argmax for one step; the argmax writes the token
        buffer the next replay embeds.  Returns (graph, tok_buffer, logits, ws)."""
        ws = self._workspace(batch)
        tok = ws["tok"]
        tok.zero_()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):         # warm-up (lazy attribute setup) outside capture
            for _ in range(2):
                lg = self._run(tok, batch, 1, states, True, ws, True)
                ops.argmax(lg, tok)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        n0 = ops.LAUNCH_COUNTER[0]
        with torch.cuda.graph(g):
            lg = self._run(tok, batch, 1, states, True, ws, True)
            ops.argmax(lg, tok)
        ops.LAUNCH_COUNTER[1] = ops.LAUNCH_COUNTER[0] - n0
        return g, tok, lg, ws

    def generate(self, prompt: torch.Tensor, n_new: int, use_graph=True):
        """Greedy generation: prompt int [B×T] → new tokens int32 [B×n_new]."""
        B = prompt.shape[0]
        lg, states = self.prefill(prompt)
        first = ops.argmax(lg)
        out = torch.empty((B, n_new), dtype=torch.int32, device=self.device)
        if n_new == 0:
            return out
        out[:, 0] = first
        if use_graph:
            g, tok, _, _ = self.capture_decode(B, states)
            # the warm-up inside capture_decode advanced the states: redo prefill
            lg, states2 = self.prefill(prompt)
            for a, b in zip(states, states2):
                a.h.copy_(b.h)
                a.conv_cache.copy_(b.conv_cache)
            tok.copy_(first)
            for i in range(1, n_new):
                g.replay()
                out[:, i] = tok
            return out
        ws = self._workspace(B)
        tok = first.clone()
        for i in range(1, n_new):
            lg = self.decode_step(tok, states, ws)
            ops.argmax(lg, tok)
            out[:, i] = tok
        return out
