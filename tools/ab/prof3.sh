#!/bin/bash
# ncu captures: cfg3 layout-T pass, cfg5 moments2d, one 8-way slab rank's pass; stage timings
mkdir -p gpurun_out
T=${TAG:-p3}
for c in cfg3 slab8 cfg2; do timeout 300 python tools/time_tail.py $c 2>&1 | tail -1 >> gpurun_out/${T}_tails.txt; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zstream -s 3 -c 1 -o gpurun_out/${T}_cfg3_zstream -f \
  python bench.py --config 3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:moments2d -s 3 -c 1 -o gpurun_out/${T}_cfg5_m2 -f \
  python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zstream -s 3 -c 1 -o gpurun_out/${T}_slab8_zstream -f \
  python tools/prof_rank.py 8 7 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_cfg3_launches.csv \
  python bench.py --config 3 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
