#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-zs19}.txt; : > $OUT
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 >> $OUT
for rep in 1 2; do for c in "cfg5 6" "1024 4" "cfg3 4" "cfg2 3"; do for l in new8 new9; do
  echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_zs.py $c 2>&1 | tail -1)" >> $OUT
done; done; done
cat $OUT
