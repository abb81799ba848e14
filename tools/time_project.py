"""Kernel timing (development aid; bench.py is the contract).

Times back-to-back calls between two events so per-call host overhead overlaps
with device work; reports the projection call alone and the full pipeline."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2012_08099_b200 import engine  # noqa: E402


def timeit(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    only = sys.argv[1] if len(sys.argv) > 1 else ""
    profile_only = len(sys.argv) > 2 and sys.argv[2] == "profile"   # (ncu A/B: time the moments-pipeline pass only)
    cases = [("cfg3-like 512^3 u16 K4", (512, 512, 512), torch.uint16, 4),
             ("cfg2 256^3 u16 K3", (256, 256, 256), torch.uint16, 3),
             ("1024^3 u16 K6", (1024, 1024, 1024), torch.uint16, 6),
             ("1024^3 u16 K4", (1024, 1024, 1024), torch.uint16, 4),
             ("1024^3 u8 K3", (1024, 1024, 1024), torch.uint8, 3),
             ("cfg5 2048^3 u16 K6", (2048, 2048, 2048), torch.uint16, 6),
             ("cfg4 1024x128^3 u8 K3", (1024, 128, 128, 128), torch.uint8, 3),
             ("cfg3 512^3 i16+1024 K4", (512, 512, 512), torch.int16, 4)]
    for name, shape, dt, K in cases:
        if only and only not in name:
            continue
        n = 1
        for d in shape:
            n *= d
        off = 0
        if dt == torch.int16:
            from paper_2012_08099_b200 import configs
            v = torch.from_numpy(configs.cfg3(0)).cuda()
            off = 1024
        elif len(shape) == 4:
            v = (torch.rand(shape, device="cuda") < 0.3).to(torch.uint8)
        elif dt == torch.uint16:
            v = engine.synth_noise(shape[2], shape[1], 0, shape[0], 5)
        else:
            v = torch.randint(0, 256, shape, dtype=torch.uint8, device="cuda")
        nbytes = v.numel() * v.element_size()
        if profile_only:
            tq = timeit(lambda: engine.project_profile(v, K, off))
            print(f"{name}: project_profile {tq:.3f} ms ({nbytes / tq / 1e6:.0f} GB/s)", flush=True)
            continue
        tp = timeit(lambda: engine.project(v, engine.num_images(K)))
        tq = timeit(lambda: engine.project_profile(v, K))
        imgs = engine.project(v, engine.num_images(K))
        t2 = timeit(lambda: engine.moments2d_images(v, imgs, K))
        tm = timeit(lambda: engine.moments(v, K))
        print(f"{name}: project {tp:.3f} ms ({nbytes / tp / 1e6:.0f} GB/s)  "
              f"project_profile {tq:.3f} ms ({nbytes / tq / 1e6:.0f} GB/s)  moments2d {t2:.3f} ms  full {tm:.3f} ms "
              f"({nbytes / tm / 1e6:.0f} GB/s, {n / tm / 1e6:.0f} GVox/s)", flush=True)
        del v
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
