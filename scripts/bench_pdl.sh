#!/bin/bash
# A/B of programmatic dependent launch per kernel class (SQ_PDL bitmask: 1 row, 2 prep, 4 ring, 8 norm, 16 gemm)
for p in ${@:-0 255 16 1 14}; do echo "SQ_PDL=$p: $(SQ_PDL=$p timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],3), round(d["config"]["step_hbm_frac"],3), "e2e", round(d["e2e"]["value"]))')"; done
