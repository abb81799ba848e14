#!/bin/bash
# bench.py (cfg5, no e2e / CPU legs) and the stage split for each lib in LIBS
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-bab}.txt; : > $OUT
for rep in 1 2; do
for l in $LIBS; do
  echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 10 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["stage_ms"])')" >> $OUT
  [ $rep = 1 ] && for c in ${TAILS:-1024k6 slab8}; do echo "$l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_tail.py $c 2>&1 | tail -1)" >> $OUT; done
done
done
cat $OUT
