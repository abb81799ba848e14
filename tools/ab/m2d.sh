#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-m2d}.txt; : > $OUT
for l in m2u8 m2u32; do DPM_LIB_PATH=tools/ab/lib_$l.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> $OUT; done
for rep in 1 2; do for l in fin m2u8 m2u32; do
  for c in 1024k6 cfg3 slab8; do echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_tail.py $c 2>&1 | tail -1)" >> $OUT; done
done; done
cat $OUT
