timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_cases.py w4a8 > gpurun_out/sanitize_w4.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_configs.py -m gpu -q -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --workload m1prefill28b --steps 5 --no-cpu-baseline > gpurun_out/bench_m1.json 2> gpurun_out/bench_m1.err
timeout 600 python bench.py --workload m1decode28b --steps 5 --no-cpu-baseline >> gpurun_out/bench_m1.json 2>> gpurun_out/bench_m1.err
