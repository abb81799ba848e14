#!/bin/bash
# Run on the GPU box (gpurun): timed bench first (must exit 0), then the ncu
# launch list and one full capture of the projection kernel on the SAME
# command.  Numbers printed under ncu are never bench values.
#   usage: tools/capture_profiles.sh TAG [CONFIG]
set -e
TAG=${1:-r01}
CFG=${2:-5}
mkdir -p gpurun_out
timeout 900 python bench.py --config "$CFG" --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > "gpurun_out/${TAG}_bench.json"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"project_stream|project_generic|moments2d|derive3d|Fill" -c 400 --csv \
  --log-file "gpurun_out/${TAG}_launches.csv" \
  python bench.py --config "$CFG" --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > "gpurun_out/${TAG}_ncu_launches.log" 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:project_stream -s 1 -c 1 \
  -o "gpurun_out/${TAG}_project_stream" -f \
  python bench.py --config "$CFG" --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > "gpurun_out/${TAG}_ncu_full.log" 2>&1
cat "gpurun_out/${TAG}_bench.json"
