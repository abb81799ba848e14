"""Per-stage device times of the moments pipeline (development aid):
projection pass, image+profile moments, epilogue -- back-to-back launches
between CUDA events, warm caches except where the input exceeds L2."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2012_08099_b200 import configs, engine  # noqa: E402


def timeit(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def graphed(fn):
    """fn captured once in a CUDA graph (no host overhead in the timing)."""
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
    torch.cuda.current_stream().wait_stream(st)
    return g.replay


def main():
    cases = {
        "cfg1": (lambda: torch.from_numpy(configs.cfg1(0)).cuda(), 3, 0),
        "cfg2": (lambda: torch.from_numpy(configs.cfg2(0)).cuda(), 3, 0),
        "cfg3": (lambda: torch.from_numpy(configs.cfg3(0)).cuda(), 4, 1024),
        "cfg4": (lambda: configs.cfg4_device(configs.cfg4_params(1024, 0), device="cuda"), 3, 0),
        "1024^3 K6": (lambda: engine.synth_noise(1024, 1024, 0, 1024, 5), 6, 0),
    }
    for name, (make, K, off) in cases.items():
        v = make()
        imgs, prof = engine.project_profile(v, K, off)
        acc = engine.moments2d_profile(v, imgs, prof, K, off)
        out = engine.derive(acc, K)
        tp = timeit(graphed(lambda: engine.project_profile(v, K, off, imgs=imgs, profile=prof)))
        tm = timeit(graphed(lambda: engine.moments2d_profile(v, imgs, prof, K, off, acc=acc)))
        td = timeit(graphed(lambda: engine.derive(acc, K, out=out)))
        g = engine.GraphedMoments(v, K, offset=off)
        tg = timeit(lambda: g.replay())
        print(f"{name}: project {tp:.1f} us  moments {tm:.1f} us  derive {td:.1f} us  graph(all) {tg:.1f} us", flush=True)
        del v, imgs, prof, acc, g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
