set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/e_pytest_gpu.log 2>&1; echo "pytest rc $?" >> gpurun_out/e_pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/e_bench_default.json 2> gpurun_out/e_bench_default.err
for c in 1 2 3 4; do timeout 600 python bench.py --config $c > gpurun_out/e_bench_cfg$c.json 2>>gpurun_out/e_bench_err.log; done
bash tools/capture_profiles.sh r01e 5
