set -x
nvidia-smi --query-gpu=name,clocks.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_zstream.py -x -q 2>&1 | tail -30
timeout 300 python tools/time_zs.py cfg5 6
DPM_LAYOUT_T_MIN_L=100000 timeout 300 python tools/time_zs.py cfg5 6
timeout 300 python tools/time_zs.py 1024 4
DPM_LAYOUT_T_MIN_L=100000 timeout 300 python tools/time_zs.py 1024 4
