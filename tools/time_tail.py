"""Per-stage device times of the streaming pipeline (development aid): the
projection graph, the 2D-moments graph with and without the fused epilogue,
and the standalone epilogue, each replayed back to back between CUDA events.
usage: python tools/time_tail.py [cfg1|cfg2|cfg3|1024k6|slab8]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2012_08099_b200 import configs, engine  # noqa: E402


def t(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


case = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
off, z0, ng = 0, 0, None
if case == "cfg1":
    vol, K = torch.from_numpy(configs.cfg1(0)).cuda(), 3
elif case == "cfg2":
    vol, K = torch.from_numpy(configs.cfg2(0)).cuda(), 3
elif case == "cfg3":
    vol, K, off = torch.from_numpy(configs.cfg3(0)).cuda(), 4, 1024
elif case == "1024k6":
    vol, K = engine.synth_noise(1024, 1024, 0, 1024, 5), 6
else:   # one rank of the 8-way cfg5 split
    vol, K, z0, ng = engine.synth_noise(2048, 2048, 1792, 256, 5), 6, 1792, 2048
a = engine.GraphedSlabStages(vol, K, offset=off, z0=z0, fused=False, n_global=ng)
b = engine.GraphedSlabStages(vol, K, offset=off, z0=z0, fused=True, n_global=ng) if ng is None else None
r = {"project": t(a.replay_project), "moments2d": t(a.replay_moments2d), "derive": t(a.replay_derive)}
if b is not None:
    r["moments2d+epilogue"] = t(b.replay_moments2d)
    g = engine.GraphedMoments(vol, K, offset=off)
    r["GraphedMoments"] = t(g.replay)
print(case, {k: round(v, 2) for k, v in r.items()}, "us")
