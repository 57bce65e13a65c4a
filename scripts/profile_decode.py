"""One eager decode step of the synthetic 8B-shaped model (few layers) for ncu launch lists."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_22879_b200 import synth  # noqa: E402
from paper_2503_22879_b200.ssm_block import Dims  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--profile", default="W4A8")
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--vocab", type=int, default=256000)
a = ap.parse_args()
d = Dims("mamba2", 4096, 8192, 128, 128, 64, 8, 4)
lm = synth.synthetic_lm(d, a.layers, a.profile, a.vocab, "cuda")
st = lm.new_states(a.batch)
ws = lm._workspace(a.batch)
tok = torch.zeros(a.batch, dtype=torch.int32, device="cuda")
for _ in range(a.steps):
    lm.decode_step(tok, st, ws)
torch.cuda.synchronize()
print("done")
