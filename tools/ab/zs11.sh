#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-zs11}.txt; : > $OUT
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 >> $OUT
for l in pf2n; do DPM_LIB_PATH=tools/ab/lib_$l.so timeout 900 python -m pytest tests/test_gpu_zstream.py -x -q 2>&1 | tail -1 >> $OUT; done
for rep in 1 2; do
  for c in "cfg5 6" "1024 6" "1024 4" "cfg3 4"; do
    for l in base new pf2n pf4n; do
      echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_zs.py $c 2>&1 | tail -1)" >> $OUT
    done
  done
done
for c in cfg3 slab8 1024k6 cfg2; do for l in base new; do echo "$l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_tail.py $c 2>&1 | tail -1)" >> $OUT; done; done
for l in base new; do echo "$l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 600 python bench.py --no-e2e --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | cut -c1-400)" >> $OUT; done
cat $OUT
