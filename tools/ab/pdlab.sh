#!/bin/bash
# PDL on/off: full GPU tests on the default build, then bench lines of every config per lib
mkdir -p gpurun_out
O=gpurun_out/${TAG:-pdl}
timeout 1500 python -m pytest tests -x -q -m gpu > ${O}_pytest.log 2>&1; echo "rc $?" >> ${O}_pytest.log
: > ${O}.txt
for rep in 1 2; do for c in 1 2 3 4 5; do for l in pdl nopdl; do
  echo "$rep cfg$c $l $(DPM_LIB_PATH=tools/ab/lib_$l.so timeout 600 python bench.py --config $c --no-e2e --no-cpu-baseline --steps 10 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["gpu_launches"], d["stage_ms"])')" >> ${O}.txt
done; done; done
for c in cfg1 cfg2 cfg3; do for l in pdl nopdl; do echo "$l $(DPM_LIB_PATH=tools/ab/lib_$l.so python tools/time_tail.py $c 2>&1 | tail -1)" >> ${O}.txt; done; done
cat ${O}.txt
