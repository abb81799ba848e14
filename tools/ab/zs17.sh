#!/bin/bash
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-zs17}.txt; : > $OUT
timeout 900 python -m pytest tests/test_gpu_zstream.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1 >> $OUT
for rep in 1 2 3; do
  for yb in 171 37 9 28 18 74; do
    echo "$rep yb$yb $(DPM_ZS_YB=$yb timeout 300 python tools/time_zs.py cfg5 6 2>&1 | tail -1)" >> $OUT
  done
done
for yb in 171 37; do
DPM_ZS_YB=$yb timeout 900 ncu --set full --clock-control none -k regex:zstream -s 1 -c 1 -o gpurun_out/zs17_yb$yb -f python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
cat $OUT
