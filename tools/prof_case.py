"""Run one projection case a few times (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2012_08099_b200 import engine  # noqa: E402

shape = tuple(int(s) for s in sys.argv[1].split("x")) if len(sys.argv) > 1 else (512, 512, 512)
K = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dt = torch.uint8 if (len(sys.argv) > 3 and sys.argv[3] == "u8") else torch.uint16
hi = 256 if dt == torch.uint8 else 65536
v = torch.randint(0, hi, shape, dtype=torch.int32, device="cuda").to(dt)
for _ in range(3):
    engine.project(v, engine.num_images(K))
torch.cuda.synchronize()
print("ok")
