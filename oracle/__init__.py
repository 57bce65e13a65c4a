"""CPU oracle for the Quamba2 quantized Mamba block path — TEST INFRASTRUCTURE ONLY.

This package is a pure-numpy restatement of the reference contract
(`/root/reference/SPEC.md` modules tensor_core, quantizer, hadamard,
ssm_block, calibrate, reorder, cli_pipeline) plus the two shipped reference
modules (`/root/reference/pkg/src/ssmquant/tensor.py`, `errors.py`).

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s `cpu_baseline` /
`--impl reference` legs may import it, and only as the checker or the timed
CPU baseline.  The product package `paper_2503_22879_b200` never imports it;
the product has no CPU fallback.

Parity pinning: the shipped reference code (`tensor.matmul`) is imported in
this container to generate `tests/golden/` fixtures (script
`tests/golden/make_golden.py`); every SPEC `[TRIVIAL]/[DERIVED]` numeric
example is a known-answer test in `tests/test_oracle_*.py`.  The hot path
itself is not shipped by the reference, so transcendental
outputs (exp/softplus/SiLU) are pinned only to the SPEC formulas
("parity partially unpinned" for those).
"""
