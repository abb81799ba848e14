"""Ad-hoc kernel timing (development aid; bench.py is the contract)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2012_08099_b200 import engine  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), sorted(ts)[len(ts) // 2]


def main():
    cases = [("cfg3-like 512^3 u16 K4", (512, 512, 512), torch.uint16, 4),
             ("cfg2 256^3 u16 K3", (256, 256, 256), torch.uint16, 3),
             ("1024^3 u16 K6", (1024, 1024, 1024), torch.uint16, 6),
             ("1024^3 u16 K4", (1024, 1024, 1024), torch.uint16, 4),
             ("1024^3 u8 K3", (1024, 1024, 1024), torch.uint8, 3),
             ("cfg5 2048^3 u16 K6", (2048, 2048, 2048), torch.uint16, 6)]
    for name, shape, dt, K in cases:
        n = shape[0] * shape[1] * shape[2]
        if dt == torch.uint16:
            v = torch.randint(0, 65536, shape, dtype=torch.int32, device="cuda").to(torch.uint16) if n < 2**31 else \
                engine.synth_noise(shape[2], shape[1], 0, shape[0], 5)
        else:
            v = torch.randint(0, 256, shape, dtype=torch.uint8, device="cuda")
        nbytes = v.numel() * v.element_size()
        tp = timeit(lambda: engine.project(v, engine.num_images(K)))
        tm = timeit(lambda: engine.moments(v, K))
        print(f"{name}: project {tp[0]:.3f} ms ({nbytes / tp[0] / 1e6:.0f} GB/s)  full {tm[0]:.3f} ms "
              f"({nbytes / tm[0] / 1e6:.0f} GB/s, {n / tm[0] / 1e6:.0f} GVox/s)", flush=True)
        del v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
