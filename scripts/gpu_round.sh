#!/bin/bash
# One GPU-box pass: parity tests, smoke, bench, launch list, ncu captures of the top kernels.
mkdir -p gpurun_out
rm -f gpurun_out/*.ncu-rep
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:state_ring -c 1 \
  -o gpurun_out/prof_ring -f python scripts/prof_kernels.py fused > gpurun_out/ncu_ring.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"prep_kernel|norm_had" -c 2 \
  -o gpurun_out/prof_prepnorm -f python scripts/prof_kernels.py fused > gpurun_out/ncu_pn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -c 2 \
  -o gpurun_out/prof_gemm -f python scripts/prof_kernels.py gemm > gpurun_out/ncu_gemm.log 2>&1
timeout 300 python scripts/bench_decode_kernels.py > gpurun_out/bdk.log 2>&1
bash scripts/bench_stages.sh > gpurun_out/stages.log 2>&1
# prefill (configs[1]): bench line, launch list, per-kernel timing, ncu of the chunk scan / conv / norm / GEMM
timeout 900 python bench.py --workload prefill27b --steps 3 > gpurun_out/bench_prefill.json 2> gpurun_out/bench_prefill.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
  --log-file gpurun_out/launches_prefill.csv python bench.py --workload prefill27b --steps 1 --warmup 3 \
  --no-cpu-baseline > gpurun_out/ncu_launch_pf.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ssd_chunk|conv1d_prefill|gate_norm" -c 3 \
  -o gpurun_out/prof_prefill -f python scripts/prof_prefill.py all 1 > gpurun_out/ncu_pf.log 2>&1
SQ_SSD_TC=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:ssd_chunk_tc -c 1 \
  -o gpurun_out/prof_ssdtc -f python scripts/prof_prefill.py ssd 1 > gpurun_out/ncu_st.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -c 2 \
  -o gpurun_out/prof_pgemm -f python scripts/prof_prefill.py gemm 1 > gpurun_out/ncu_pg.log 2>&1
(timeout 300 python scripts/prof_prefill.py all 3; SQ_SSD_TC=1 timeout 300 python scripts/prof_prefill.py ssd 3 | sed 's/^ssd/ssd_tcgen05/'; \
  timeout 300 python scripts/prof_prefill.py gemm 3) > gpurun_out/prefill_kernels.txt 2>&1
for w in decode8b_w4a16 m1prefill28b m1decode28b; do timeout 600 python bench.py --workload $w --steps 5; done > gpurun_out/bench_other.json 2>/dev/null
echo done
