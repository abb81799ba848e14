#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-zs14}.txt; : > $OUT
for l in new4 fbo; do DPM_LIB_PATH=tools/ab/lib_$l.so timeout 900 python -m pytest tests/test_gpu_zstream.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> $OUT; done
for rep in 1 2; do
  for c in "cfg5 6" "1024 6" "1024 4" "cfg3 4" "cfg2 3"; do
    for l in new3 new4 fbo; do
      echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_zs.py $c 2>&1 | tail -1)" >> $OUT
    done
  done
done
for c in slab8; do for l in new3 new4 fbo; do echo "$l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_tail.py $c 2>&1 | tail -1)" >> $OUT; done; done
cat $OUT
