#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench, launch list, ncu captures of the top kernels.
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:state_update -c 2 \
  -o gpurun_out/prof_state -f python scripts/prof_kernels.py state > gpurun_out/ncu_state.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm -c 2 \
  -o gpurun_out/prof_gemm -f python scripts/prof_kernels.py gemm > gpurun_out/ncu_gemm.log 2>&1
timeout 600 python scripts/bench_gemm.py > gpurun_out/bench_gemm.log 2>&1
echo done
