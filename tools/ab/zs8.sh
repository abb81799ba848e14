timeout 900 python -m pytest tests/test_gpu_zstream.py -x -q 2>&1 | tail -2
DPM_LIB_PATH=tools/ab/lib_nw8.so timeout 900 python -m pytest tests/test_gpu_zstream.py -x -q 2>&1 | tail -2
for c in "cfg5 6" "1024 6" "1024 4" "cfg3 4" "cfg2 3"; do
  timeout 300 python tools/time_zs.py $c
  DPM_LIB_PATH=tools/ab/lib_nw8.so timeout 300 python tools/time_zs.py $c | sed 's/^/nw8: /'
done
DPM_LIB_PATH=tools/ab/lib_nw8.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:zstream -s 2 -c 1 -o gpurun_out/zs8 -f python tools/prof_zs.py 1024x1024x1024 6 > gpurun_out/zs8_ncu.log 2>&1
