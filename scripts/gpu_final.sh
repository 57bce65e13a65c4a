#!/bin/bash
# Round-end GPU evidence: full GPU tests, default bench (decode + prefill sub-record), the other
# BASELINE configs, the decode launch list, compute-sanitizer.  gpurun -- bash scripts/gpu_final.sh
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for w in decode8b_w4a16 m1prefill28b m1decode28b; do
  timeout 600 python bench.py --workload $w --steps 10 --no-cpu-baseline >> gpurun_out/bench_other.json 2>> gpurun_out/bench_other.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -s 2000 -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-prefill > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
bash scripts/sanitize.sh
