# one GPU round: tests, smoke, default bench (cfg5), configs 1-4, profiles of cfg5
TAG=${TAG:-r01}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/${TAG}_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench_cfg5.json 2> gpurun_out/${TAG}_bench_cfg5.err
if [ -z "$SKIP_CFGS" ]; then
  for c in 1 2 3 4; do timeout 600 python bench.py --config $c > gpurun_out/${TAG}_bench_cfg$c.json 2>>gpurun_out/${TAG}_bench_err.log; done
fi
bash tools/capture_profiles.sh ${TAG} 5
