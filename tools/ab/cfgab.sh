#!/bin/bash
# bench lines of CFGS for each lib in LIBS (two interleaved repetitions) + stage split
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-cab}.txt; : > $OUT
for rep in 1 2; do for c in ${CFGS:-2 3}; do for l in $LIBS; do
  echo "$rep cfg$c $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["stage_ms"])')" >> $OUT
done; done; done
for c in ${TAILS:-cfg2 cfg3}; do for l in $LIBS; do echo "$l $(DPM_LIB_PATH=tools/ab/lib_$l.so python tools/time_tail.py $c 2>&1 | tail -1)" >> $OUT; done; done
cat $OUT
