timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "direct" 2>&1 | tail -3
cd baseline/_ref_tests && PYTHONPATH=$GRAFT_REPO_ROOT timeout 1200 python -m pytest . -q -p no:cacheprovider -rfE --continue-on-collection-errors --tb=line 2>&1 | grep -E "^/|^E |^FAILED|^ERROR|passed|failed" | head -60
