#!/bin/bash
# repeat the layout-T / parity tests (timing-dependent hazards), then memcheck small passes
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-stress}.txt; : > $OUT
for i in 1 2 3; do timeout 900 python -m pytest tests/test_gpu_zstream.py tests/test_gpu_parity.py tests/test_gpu_fused.py -x -q 2>&1 | tail -1 >> $OUT; done
cat > /tmp/mc.py <<'PY'
import numpy as np, torch, sys
sys.path.insert(0, ".")
import oracle
import paper_2012_08099_b200 as vm
from paper_2012_08099_b200 import engine
rng = np.random.default_rng(5)
for shape, dt, order in (((20, 30, 520), np.uint16, 6), ((17, 14, 264), np.uint16, 4), ((12, 26, 256), np.uint8, 3), ((9, 13, 200), np.uint16, 5), ((6, 20, 128), np.uint8, 3)):
    vol = rng.integers(0, np.iinfo(dt).max + 1, size=shape).astype(dt)
    res = engine.moments(torch.from_numpy(vol).cuda(), order)
    torch.cuda.synchronize()
    want = oracle.dpm(vol, order)
    assert engine.i128_to_ints(res.i128[0].cpu().numpy()) == [want[k] for k in vm.moment_indices(order)], shape
print("memcheck cases ok")
PY
timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python /tmp/mc.py > gpurun_out/${TAG:-stress}_memcheck.log 2>&1; echo "memcheck rc $?" >> $OUT
DPM_ZS_XT_MAJOR_MB=0 DPM_ZS_YB=2 timeout 1500 compute-sanitizer --tool memcheck --error-exitcode 9 python /tmp/mc.py > gpurun_out/${TAG:-stress}_memcheck_yb2.log 2>&1; echo "memcheck yb2 rc $?" >> $OUT
tail -3 gpurun_out/${TAG:-stress}_memcheck.log >> $OUT
cat $OUT
