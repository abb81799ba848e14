#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-zs12}.txt; : > $OUT
for l in $LIBS; do [ $l = base ] && continue; DPM_LIB_PATH=tools/ab/lib_$l.so timeout 900 python -m pytest tests/test_gpu_zstream.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> $OUT; done
IFS='|' read -ra CS <<< "${CASES:-cfg5 6|1024 6|1024 4|cfg3 4}"
for rep in 1 2; do
  for c in "${CS[@]}"; do
    for l in $LIBS; do
      echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_zs.py $c 2>&1 | tail -1)" >> $OUT
    done
  done
done
cat $OUT
