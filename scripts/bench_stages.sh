#!/bin/bash
# In-graph time of each decode-step launch alone (SQ_DECODE_STAGES bitmask), b=64, 8B shape.
for m in 7 1 2 4; do
  echo "stages=$m: $(SQ_DECODE_STAGES=$m python scripts/bench_decode_kernels.py 2>&1 | grep decode_step)"
done
