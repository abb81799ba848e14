#!/bin/bash
# ncu launch lists (kernel durations) of the bench step for configs 1-4 (GPU box)
mkdir -p gpurun_out
for c in ${CFGS:-1 2 3 4}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/${TAG:-ll}_cfg${c}_launches.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG:-ll}_cfg${c}_ncu.log 2>&1
done
