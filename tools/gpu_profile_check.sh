mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/p_pytest.log 2>&1; echo "rc $?" >> gpurun_out/p_pytest.log
timeout 600 python tools/time_project.py > gpurun_out/p_time.log 2>&1
