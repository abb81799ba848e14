timeout 900 python -m pytest tests/test_gpu_zstream.py -x -q 2>&1 | tail -3
timeout 300 python tools/time_zs.py cfg5 6
DPM_LAYOUT_T_MIN_L=100000 timeout 300 python tools/time_zs.py cfg5 6
timeout 300 python tools/time_zs.py 1024 4
timeout 300 python tools/time_zs.py cfg3 4
DPM_LAYOUT_T_MIN_L=100000 timeout 300 python tools/time_zs.py cfg3 4
timeout 600 ncu --set full --clock-control none --import-source on -k regex:zstream -s 2 -c 1 -o gpurun_out/zs3 -f python tools/prof_zs.py 1024x1024x1024 6 > gpurun_out/zs3_ncu.log 2>&1
