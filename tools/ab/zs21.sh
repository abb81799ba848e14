#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-zs21}.txt; : > $OUT
for rep in 1 2; do for l in new8 new8b new9 new9p; do
  echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_zs.py cfg3 4 2>&1 | tail -1)" >> $OUT
done; done
cat $OUT
