#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-m2c}.txt; : > $OUT
for rep in 1 2; do for l in fin m2t16 m2t32 m2b5; do
  echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["stage_ms"])')" >> $OUT
  echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_tail.py 1024k6 2>&1 | tail -1)" >> $OUT
done; done
for l in fin m2t16; do echo "$l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_tail.py slab8 2>&1 | tail -1)" >> $OUT; done
for c in 3 2 1; do echo "cfg$c $(timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])')" >> $OUT; done
cat $OUT
