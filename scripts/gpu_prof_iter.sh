timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-prefill > /dev/null 2>&1
python scripts/launch_table.py gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mamba1_scan_staged -c 1 -o gpurun_out/prof_m1scan -f python bench.py --workload m1prefill28b --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_m1.log 2>&1
