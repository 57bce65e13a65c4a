#!/bin/bash
# Quick GPU pass: GPU tests (optionally a subset) + GEMM timings + bench + launch list.
mkdir -p gpurun_out
SEL=${1:-tests}
timeout 1200 python -m pytest $SEL -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python scripts/bench_gemm.py > gpurun_out/bench_gemm.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo done
