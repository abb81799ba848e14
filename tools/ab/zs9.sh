#!/bin/bash
# early stage release / producer placement / z-chunked run order: tests, then interleaved timings
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-zs9}.txt; : > $OUT
for l in ${LIBS:-erel0 erel1 erel2}; do
  echo "== tests $l" >> $OUT
  DPM_LIB_PATH=tools/ab/lib_$l.so timeout 900 python -m pytest tests/test_gpu_zstream.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2 >> $OUT
done
echo "== tests base ZH=2" >> $OUT
DPM_ZS_ZH=2 DPM_LIB_PATH=tools/ab/lib_base.so timeout 900 python -m pytest tests/test_gpu_zstream.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2 >> $OUT
for rep in 1 2; do
  for c in "cfg5 6" "1024 6" "1024 4" "cfg3 4"; do
    for l in base ${LIBS:-erel0 erel1 erel2}; do
      for zh in ${ZHS:-1 2 4}; do
        echo "$rep $l zh$zh $(DPM_ZS_ZH=$zh DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_zs.py $c 2>&1 | tail -1)" >> $OUT
      done
    done
  done
done
cat $OUT
