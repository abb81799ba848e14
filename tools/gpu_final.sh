#!/bin/bash
# Round-end evidence run (GPU box): tests, smoke, every bench line, the
# reference arm, the simulated per-rank split, launch lists and ncu captures.
TAG=${TAG:-r02c}
mkdir -p gpurun_out
O=gpurun_out/$TAG
timeout 1500 python -m pytest tests -x -q -m gpu > ${O}_pytest_gpu.log 2>&1; echo "pytest rc $?" >> ${O}_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > ${O}_smoke.log 2>&1; echo "smoke rc $?" >> ${O}_smoke.log
timeout 1200 python bench.py > ${O}_bench_cfg5.json 2> ${O}_bench_cfg5.err
for c in 1 2 3 4; do timeout 900 python bench.py --config $c > ${O}_bench_cfg$c.json 2>> ${O}_bench_err.log; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > ${O}_bench_reference_cfg5.json 2>> ${O}_bench_err.log
for g in 2 4 8; do timeout 900 python bench.py --simulate-ranks $g --steps 5 >> ${O}_simulate_ranks_cfg5.jsonl 2>> ${O}_bench_err.log; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${O}_cfg5_launches.csv \
  python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fused|zero_kernel|moments2d|derive" -c 60 --csv --log-file ${O}_cfg4_launches.csv \
  python bench.py --config 4 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:zstream -s 1 -c 1 -o ${O}_cfg5_zstream -f \
  python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o ${O}_cfg4_fused -f \
  python bench.py --config 4 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
echo done
