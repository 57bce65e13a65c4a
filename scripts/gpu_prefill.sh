#!/bin/bash
# Prefill iteration pass: kernel tests, per-kernel timing, optional ncu capture of one kernel.
#   bash scripts/gpu_prefill.sh [ncu-kernel-regex] [prof_prefill mode]
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_model.py -m gpu -q -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/prof_prefill.py all 5 > gpurun_out/prefill_kernels.txt 2>&1; cat gpurun_out/prefill_kernels.txt
if [ -n "$1" ]; then
  timeout 900 ncu --set full --import-source on --clock-control none -k "regex:$1" -c 1 -o gpurun_out/prof_pf -f \
    python scripts/prof_prefill.py ${2:-all} 1 > gpurun_out/ncu_pf.log 2>&1; tail -2 gpurun_out/ncu_pf.log
fi
timeout 600 python bench.py --workload prefill27b --no-cpu-baseline --steps 3 > gpurun_out/bench_pf.json 2> gpurun_out/bench_pf.err; cat gpurun_out/bench_pf.json
