#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-zs15}.txt; : > $OUT
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 >> $OUT
for rep in 1 2; do
  for c in "cfg5 6" "1024 6" "1024 4" "cfg3 4" "cfg2 3"; do
    for l in new4 new5; do
      echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_zs.py $c 2>&1 | tail -1)" >> $OUT
    done
  done
done
for c in slab8 cfg3; do for l in new4 new5; do echo "$l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_tail.py $c 2>&1 | tail -1)" >> $OUT; done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zstream -s 1 -c 1 -o gpurun_out/zs15_cfg5 -f python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zstream -s 3 -c 1 -o gpurun_out/zs15_cfg3 -f python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
cat $OUT
