timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused -s 3 -c 1 -o gpurun_out/ab3_cfg1_fused -f python bench.py --config 1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:moments2d -s 3 -c 1 -o gpurun_out/ab3_cfg2_m2 -f python bench.py --config 2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
TAG=ab3 LIBS="base idp" CASES="cfg5 6|1024 6|1024 4" bash tools/ab/zsab.sh
