"""In-graph marginal cost of each launch class of the Mamba2-8B W4A8 b=64 decode step: the step
graph is re-captured with one class replaced by nothing (outputs become garbage, timing stays
valid) and the per-step difference is that class's marginal cost, PDL overlap included.
usage: python scripts/ablate_decode.py [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import ops, synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import DeviceLinear, Dims  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dev = "cuda"
d = Dims("mamba2", 4096, 8192, 128, 128, 64, 8, 4)
lm = synth.synthetic_lm(d, 56, "W4A8", 256000, dev)
B = 64
states = lm.new_states(B)
for s in states:
    s.h.random_(-100, 100)


def timed():
    g, tok, _, _ = lm.capture_decode(B, states)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3   # us per step


base = timed()
print(f"full step {base:9.1f} us  ({B / base * 1e6:8.0f} tok/s)", flush=True)
orig_a8 = DeviceLinear.a8
head = lm.head


def skip_if(pred):
    def a8(self, a_codes, epi, out=None, col_scale=None):
        if pred(self):
            return out if out is not None else torch.empty((a_codes.shape[0], self.N), device=a_codes.device)
        return orig_a8(self, a_codes, epi, out, col_scale)
    return a8


for name, pred in [("in_proj", lambda s: s.N == d.in_proj_out), ("out_proj", lambda s: s.N == d.d_model and s is not head),
                   ("head", lambda s: s is head)]:
    DeviceLinear.a8 = skip_if(pred)
    t = timed()
    DeviceLinear.a8 = orig_a8
    per = (base - t) / (56 if name != "head" else 1)
    print(f"without {name:9s} {t:9.1f} us  -> marginal {base - t:8.1f} us/step = {per:7.2f} us per launch", flush=True)
orig_dec = ops.mamba2_decode_step_int8
ops.mamba2_decode_step_int8 = lambda p, B, zx, cc, st, yq=None, y=None, ws=None, gsum=None: yq
t = timed()
ops.mamba2_decode_step_int8 = orig_dec
print(f"without ssm-step  {t:9.1f} us  -> marginal {base - t:8.1f} us/step = {(base - t) / 56:7.2f} us per layer", flush=True)
orig_rn = ops.rmsnorm_quant
ops.rmsnorm_quant = lambda x, gamma, eps, s, out=None, gsum=None: out
t = timed()
ops.rmsnorm_quant = orig_rn
print(f"without rmsnorm   {t:9.1f} us  -> marginal {base - t:8.1f} us/step = {(base - t) / 57:7.2f} us per launch", flush=True)
