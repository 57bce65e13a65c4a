#!/bin/bash
# ncu --set full captures inside the default bench's replayed decode step (steady state, every
# layer's state and weights streaming from HBM): one layer's decode SSM kernels (prep, state ring,
# norm) and its two W4A8 GEMMs.  Then: python scripts/summarize_profiles.py <tag>
mkdir -p gpurun_out/prof
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"prep_kernel|state_ring_kernel|norm_had8192" \
  -s 600 -c 3 -f -o gpurun_out/prof/prof_ring python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-prefill \
  > gpurun_out/prof/ncu_ring.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_w4a8_pg" \
  -s 400 -c 2 -f -o gpurun_out/prof/prof_gemm python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-prefill \
  > gpurun_out/prof/ncu_gemm.log 2>&1
