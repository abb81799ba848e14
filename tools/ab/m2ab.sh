timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/m2_pytest.log 2>&1; echo "rc $?" >> gpurun_out/m2_pytest.log
TAG=m2ab LIBS="m2old m2loc" TAILS="slab8 1024k6 cfg3 cfg2" bash tools/ab/benchab.sh
