#!/bin/bash
# ncu capture of one fused decode step (8B shapes, B=64): gpurun -- bash scripts/gpu_prof_fused.sh
python scripts/prof_fused.py > gpurun_out/prof_fused.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -f -o gpurun_out/fused \
  python scripts/prof_fused.py >> gpurun_out/prof_fused.txt 2>&1
