timeout 900 python -m pytest tests/test_gpu_cfg4.py tests/test_gpu_profile.py -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
