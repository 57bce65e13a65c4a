#!/bin/bash
for d in ${GDBG:-2}; do echo "== SQ_GEMM_DBG=$d (2 timeline, +4 no tmem st, +32 no main-loop MMA)"; SQ_GEMM_DBG=$d python scripts/prof_kernels.py gemm 2>&1 | grep "cta 0" | tail -8; done
