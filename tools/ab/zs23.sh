#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-zs23}.txt; : > $OUT
for rep in 1 2; do for c in "cfg5 6" "1024 6" "1024 5" "1024 4" "1024 3" "cfg3 4" "cfg3 3" "cfg2 3" "cfg2 4" "cfg2 6"; do for l in fin pdl0; do
  echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_zs.py $c 2>&1 | tail -1)" >> $OUT
done; done; done
for c in 1 2 3 4; do for l in fin pdl0; do
  echo "cfg$c $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')" >> $OUT
done; done
cat $OUT
