"""Drop-in e2e timing of dpm_moments(Volume(numpy)) on the cfg5 volume for the
current uploader settings (DPM_UPLOAD_THREADS / DPM_UPLOAD_CHUNK_MB); dev aid."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2012_08099_b200 as vm  # noqa: E402
from paper_2012_08099_b200 import engine  # noqa: E402

host = engine.synth_noise(2048, 2048, 0, 2048, 5).cpu().numpy()
v = vm.Volume(host)
vm.dpm_moments(v, 6)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    vm.dpm_moments(v, 6)
    ts.append(time.perf_counter() - t0)
print(f"threads {os.environ.get('DPM_UPLOAD_THREADS', '8')} chunk {os.environ.get('DPM_UPLOAD_CHUNK_MB', '64')} MB: "
      f"{[round(t, 3) for t in ts]} s -> {host.size / min(ts) / 1e9:.1f} GVoxel/s (best), cores {os.cpu_count()}")
