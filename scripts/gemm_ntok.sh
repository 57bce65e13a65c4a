#!/bin/bash
# Prefill W8A8 GEMM time vs forced token tile (SQ_GEMM_NTOK), 2.7B in_proj / out_proj shapes.
for n in 0 128 256; do echo "SQ_GEMM_NTOK=$n: $(SQ_GEMM_NTOK=$n timeout 300 python scripts/prof_prefill.py gemm 5 2>&1 | tail -1)"; done
