#!/bin/bash
# One GPU round (round 2): tests, smoke, bench of every config, cfg5 launch
# list and one full ncu capture of the cfg5 projection kernel.
TAG=${TAG:-r02b}
mkdir -p gpurun_out
python -c "import torch; print(torch.cuda.get_device_name(0))" > gpurun_out/${TAG}_dev.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/${TAG}_pytest_gpu.log
  timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/${TAG}_smoke.log
fi
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${TAG}_bench_cfg5.json 2> gpurun_out/${TAG}_bench_cfg5.err
for c in ${CFGS:-1 2 3 4}; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${TAG}_bench_cfg$c.json 2>>gpurun_out/${TAG}_bench_err.log; done
CFG=${PCFG:-5}
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file "gpurun_out/${TAG}_cfg${CFG}_launches.csv" \
  python bench.py --config "$CFG" --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > "gpurun_out/${TAG}_ncu_launches.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-project_stream|zstream}" -s 2 -c 1 \
  -o "gpurun_out/${TAG}_cfg${CFG}_top" -f \
  python bench.py --config "$CFG" --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > "gpurun_out/${TAG}_ncu_full.log" 2>&1
echo done
