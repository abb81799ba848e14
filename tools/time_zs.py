"""A/B timing of the moments pipeline's projection pass (development aid):
project_profile on a device-resident volume, back-to-back graph replays
between CUDA events.  Usage: python tools/time_zs.py [cfg5|1024|cfg3|cfg2] [order]
(DPM_LAYOUT_T_MIN_L=100000 in the environment forces the classic layout)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2012_08099_b200 import configs, engine  # noqa: E402


def graphed(fn):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
    torch.cuda.current_stream().wait_stream(st)
    return g.replay


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
    return e0.elapsed_time(e1) / reps


def main():
    case = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
    order = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    offset = 0
    if case == "cfg5":
        vol = engine.synth_noise(2048, 2048, 0, 2048, 5)
    elif case == "1024":
        vol = engine.synth_noise(1024, 1024, 0, 1024, 5)
    elif case == "cfg3":
        vol = torch.from_numpy(configs.cfg3()).cuda()
        offset = 1024
    else:
        vol = torch.from_numpy(configs.cfg2()).cuda()
    nbytes = vol.numel() * vol.element_size()
    kind = engine.acc_kind(vol, order, offset)
    imgs, prof = engine.project_profile(vol, order, offset=offset)
    ms = timeit(graphed(lambda: engine.project_profile(vol, order, offset=offset, imgs=imgs, profile=prof)))
    full = engine.GraphedMoments(vol, order, offset=offset)
    ms_full = timeit(full.replay)
    print(f"{case} order {order} layout {kind}: projection(+zeroing) {ms:.4f} ms = {nbytes / ms / 1e6:.0f} GB/s;"
          f" full pipeline {ms_full:.4f} ms = {nbytes / ms_full / 1e6:.0f} GB/s "
          f"({vol.numel() / ms_full / 1e6:.0f} GVoxel/s), status {int(full.out.status[0])}")


if __name__ == "__main__":
    main()
