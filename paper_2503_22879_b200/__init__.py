"""B200-native (sm_100a) implementation of Quamba2's quantized Mamba block forward path.

Host API mirrors the reference package `ssmquant` (SPEC.md module names); the hot path
runs in libssmquant_sm100.so (hand-written CUDA, C-ABI in include/ssmquant_sm100.h).
The top-level `ssmquant` package in this repo re-exports these modules under the
reference names.
"""
__version__ = "0.1.0"
