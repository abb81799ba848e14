#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-zs16}.txt; : > $OUT
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -2 >> $OUT
for c in "1024^3 u16 K6" "1024^3 u16 K4" "1024^3 u8 K3" "cfg2"; do for l in new6 new7; do echo "$l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 300 python tools/time_project.py "$c" 2>&1 | tail -1)" >> $OUT; done; done
cat $OUT
