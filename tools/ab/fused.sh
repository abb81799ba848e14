#!/bin/bash
# fused small-volume pass: parity tests, then config 1 / 4 bench lines for the
# default build and the 8-warp variant, and one ncu capture of the cfg4 kernel
mkdir -p gpurun_out
T=${TAG:-fb}
timeout 900 python -m pytest tests/test_gpu_fused.py tests/test_gpu_cfg4.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo "rc $?" >> gpurun_out/${T}_tests.log
for c in 4 1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench_cfg$c.json 2>>gpurun_out/${T}_err.log
  DPM_LIB_PATH=tools/ab/lib_fb8.so timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench8_cfg$c.json 2>>gpurun_out/${T}_err.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${T}_cfg4_launches.csv \
  python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o gpurun_out/${T}_cfg4_fused -f \
  python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1
tail -3 gpurun_out/${T}_tests.log
