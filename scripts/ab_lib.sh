#!/bin/bash
# Same-box A/B of two builds of the library on the decode bench: ab/lib_head.so vs ab/lib_new.so
L=paper_2503_22879_b200/libssmquant_sm100.so
for r in 1 2; do for v in head new; do
  cp ab/lib_$v.so $L
  echo "$v: $(timeout 300 python bench.py --no-cpu-baseline ${@} 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],3))')"
done; done
cp ab/lib_new.so $L
