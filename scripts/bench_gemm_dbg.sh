#!/bin/bash
for d in 0 1; do echo "SQ_GEMM_DBG=$d"; SQ_GEMM_DBG=$d python scripts/bench_decode_kernels.py 2>&1 | grep -E "proj"; done
