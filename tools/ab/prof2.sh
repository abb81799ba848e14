python bench.py --config 5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:zstream -s 1 -c 1 -o gpurun_out/p2_cfg5_zs -f python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:moments2d -s 1 -c 1 -o gpurun_out/p2_cfg5_m2 -f python bench.py --config 5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
