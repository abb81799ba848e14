#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-zs20}.txt; : > $OUT
for rep in 1 2 3; do for l in new8 new9; do
  echo "$rep $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_zs.py cfg3 4 2>&1 | tail -1)" >> $OUT
done; done
for l in new8 new9; do
DPM_LIB_PATH=tools/ab/lib_$l.so timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum --clock-control none -k regex:zstream -c 6 --csv --log-file gpurun_out/zs20_$l.csv python tools/time_zs.py cfg3 4 > /dev/null 2>&1
done
cat $OUT
