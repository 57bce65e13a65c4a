#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the small-shape kernel cases
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for c in w4a8 w8a8 decode ssd w4a16 m1; do
    echo "== $tool $c"
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py $c 2>&1 | tail -8
  done
done > gpurun_out/sanitize.txt 2>&1
