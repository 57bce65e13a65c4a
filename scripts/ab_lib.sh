#!/bin/bash
# Same-box A/B of library builds on the decode bench: every ab/lib_*.so, two passes
L=paper_2503_22879_b200/libssmquant_sm100.so
cp $L /tmp/lib_orig.so
for r in 1 2; do for f in ab/lib_*.so; do
  cp $f $L
  echo "$(basename $f .so): $(timeout 300 python bench.py --no-cpu-baseline ${@} 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]), round(d["ms_per_step"],3))')"
done; done
cp /tmp/lib_orig.so $L
