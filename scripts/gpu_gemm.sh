#!/bin/bash
# GEMM iteration pass: timeline of CTA 0, isolated in-graph kernel times, decode bench.
mkdir -p gpurun_out
bash scripts/gemm_timeline.sh 2>&1 | tail -5
timeout 300 python scripts/bench_decode_kernels.py 2>&1 | grep -E "proj|decode_step"
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; cut -c1-200 gpurun_out/bench.json
