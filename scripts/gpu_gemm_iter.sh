timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -rf -k "gemm" > gpurun_out/pytest_gemm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gemm.log
python scripts/probe_w4.py base > gpurun_out/probe.txt 2>&1
python scripts/probe_tl.py tl > gpurun_out/probe_tl.txt 2>&1
python scripts/bench_gemm.py > gpurun_out/bench_gemm.txt 2>&1
