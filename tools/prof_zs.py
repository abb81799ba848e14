"""Run the moments pipeline's projection pass a few times (for ncu captures).
Usage: python tools/prof_zs.py LxMxN order [u8|u16]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2012_08099_b200 import engine  # noqa: E402

l, m, n = (int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "1024x1024x1024").split("x"))
K = int(sys.argv[2]) if len(sys.argv) > 2 else 6
if len(sys.argv) > 3 and sys.argv[3] == "u8":
    v = torch.randint(0, 256, (n, m, l), dtype=torch.int32, device="cuda").to(torch.uint8)
else:
    v = engine.synth_noise(l, m, 0, n, 5)
for _ in range(3):
    engine.project_profile(v, K)
torch.cuda.synchronize()
print("ok", engine.acc_kind(v, K))
