#!/bin/bash
# GEMM iteration: W4A8/W8A8 kernel parity tests, projection timings, one ncu capture of the in_proj W4A8 GEMM.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -rf -k "gemm" > gpurun_out/pytest_gemm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gemm.log
timeout 300 python scripts/bench_gemm.py > gpurun_out/bench_gemm.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_w4a8 -s 2 -c 1 -o gpurun_out/prof_w4in -f python scripts/prof_gemm.py in w4a8 > gpurun_out/ncu_w4in.log 2>&1
