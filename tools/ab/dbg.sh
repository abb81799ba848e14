DPM_DEBUG=1 CUDA_LAUNCH_BLOCKING=1 timeout 300 python tools/ab/dbg.py 2>&1 | tail -8
