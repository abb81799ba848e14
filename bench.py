#!/usr/bin/env python
"""bench.py -- the DPM hot path on B200: one JSON line (driver contract).

Workload (default, ``--config 5``): BASELINE.json config 5, one 2048^3 uint16
volume (16 GiB) of seeded smooth noise, all raw 3D moments up to order 6.
At N GPUs the volume is z-slab sharded (each rank generates and holds only
its planes); a step = project the slab -> exact 2D moments in global
coordinates -> NCCL all-reduce of the 2D-moment limbs -> device epilogue.
The volume (16 GiB) is far larger than L2 (126 MB), so no L2 flush is needed
between steps.

Reported keys beyond the base contract:
  roofline      projection-stage bytes/s vs the measured HBM copy peak
                (MEASURED_PEAKS.json), plus ncu DRAM traffic per launch from
                profiles/ when a capture for this workload is committed
  cpu_baseline  the C restatement of the reference algorithm (oracle/,
                OpenMP) timed on this host on a bounded slab of the same data
  e2e           the same metric through the public host-buffer API
                (paper_2012_08099_b200.streaming: pinned host -> chunked H2D
                overlapped with the projection pass -> result D2H)
  clocks        SM clock / throttle reasons sampled during the timed region
``--impl reference`` times the CPU port of the reference path instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG_DESC = {
    1: "cfg1: 64^3 uint8 i.i.d. uniform (seed 0), order 3",
    2: "cfg2: 256^3 uint16 MRI-like phantom (seed 0), order 3",
    3: "cfg3: 512^3 int16 CT-like (+1024 offset on device), order 4",
    4: "cfg4: 1024 x 128^3 binary uint8 rotated ellipsoids, order 3, batch-sharded",
    5: "cfg5: 2048^3 uint16 smooth lattice noise (16 GiB, seed 5), order 6, z-slab-sharded",
}
CFG5_SEED = 5
ORDER = {1: 3, 2: 3, 3: 4, 4: 3, 5: 6}
TOTAL_VOXELS = {1: 64 ** 3, 2: 256 ** 3, 3: 512 ** 3, 4: 1024 * 128 ** 3, 5: 2048 ** 3}


def workload_config(cfg: int, world: int, cache: str) -> dict:
    """The ``config`` object of the JSON line -- identical for both arms."""
    par = {5: f"z-slab x{world}", 4: f"batch x{world}"}.get(cfg, f"replicas x{world}")
    total = TOTAL_VOXELS[cfg] * (world if cfg in (1, 2, 3) else 1)
    return {"workload": CONFIG_DESC[cfg], "order": ORDER[cfg], "parallelism": par, "voxels_per_step": total,
            "cache": cache}


def cache_note(cfg: int) -> str:
    return ("inputs larger than L2 (no flush)" if cfg in (3, 4, 5)
            else "L2 scrubbed before every step (untimed 2xL2 write), per-step events")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--simulate-ranks", type=int, default=0, metavar="G",
                    help="cfg5 only: time, on this one GPU, the per-rank step of each of the G ranks of the "
                         "G-way z-slab split (slab of N/G planes at its global z0, epilogue as its own stage) "
                         "and predict the G-GPU figure (no all-reduce is run)")
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    def __init__(self, index: int):
        self.index = index
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                getattr(pynvml, "nvmlClocksThrottleReasonHwSlowdown", 0x8): "hw_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
                getattr(pynvml, "nvmlClocksThrottleReasonSwPowerCap", 0x4): "sw_power_cap",
                getattr(pynvml, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake",
            }

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
                        for bit, name in names.items():
                            if r & bit:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    self._stop.wait(0.02)

            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            pass
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def ncu_traffic(workload_key: str):
    """DRAM bytes per projection launch from a committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(workload_key)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# CPU baselines.  ``oracle/`` holds the exact C restatement of the reference
# path (the "port", OpenMP on every host thread); ``oracle.reference`` loads
# the reference package itself (numpy, single-threaded by design) from the
# driver's offline install baseline/_ref when it is present.

def cpu_sample(cfg: int, kind: str):
    """A bounded sample of the workload for one CPU leg: (volumes, order, offset, description).
    kind: "port" (the C port of dpm_moments), "naive" (the C port of naive_moments),
    "ref_dpm" / "ref_naive" (the reference's own numpy engines; orders <= 4)."""
    from paper_2012_08099_b200 import configs as synth
    import oracle
    order, offset = ORDER[cfg], (1024 if cfg == 3 else 0)
    if kind in ("ref_dpm", "ref_naive"):
        order = min(order, 4 if kind == "ref_dpm" else 3)   # the reference accepts orders 3-4; naive at 2048 wide overflows at 4
    if cfg == 5:
        planes = {"port": 32, "naive": 1, "ref_dpm": 16, "ref_naive": 2}[kind]
        v = oracle.synth_noise(2048, 2048, 0, planes, CFG5_SEED)
        return [v], order, 0, f"planes 0-{planes - 1} of the cfg5 volume (2048x2048x{planes}), order {order}"
    if cfg == 4:
        n = {"port": 16, "naive": 1, "ref_dpm": 8, "ref_naive": 2}[kind]
        p = synth.cfg4_params(n, 0)
        return [synth.cfg4_volume_numpy(p[i]) for i in range(n)], order, 0, f"{n} of the 1024 cfg4 volumes, order {order}"
    if cfg == 3:
        v = synth.cfg3(0)
        if kind in ("naive", "ref_naive"):
            v = v[:8]
            return [v], order, offset, f"planes 0-7 of the cfg3 volume (512x512x8), order {order}"
        return [v], order, offset, f"the whole cfg3 volume, order {order}"
    v = synth.cfg2(0) if cfg == 2 else synth.cfg1(0)
    if cfg == 2 and kind in ("naive", "ref_naive"):
        v = v[:16]
        return [v], order, 0, f"planes 0-15 of the cfg2 volume (256x256x16), order {order}"
    return [v], order, 0, f"the whole cfg{cfg} volume, order {order}"


def _as_u16(v, offset):
    return (v.astype(np.int32) + offset).astype(np.uint16) if offset else v


def cpu_leg(cfg: int, kind: str, budget_s: float) -> dict:
    """Time one CPU leg: the ports with the oracle's own loop on every host
    thread, the reference engines with the reference's own best-of-R protocol
    (harness._time_best_of, harness.py:187-204) on its single core."""
    import oracle
    vols, order, offset, sample = cpu_sample(cfg, kind)
    nvox = sum(int(np.prod(v.shape)) for v in vols)
    if kind in ("port", "naive"):
        threads = os.cpu_count() or 1
        oracle.set_threads(threads)
        fn = oracle.dpm if kind == "port" else oracle.naive_direct

        def call():
            for v in vols:
                fn(v, order, offset=offset)
        call()
        reps, t0 = 0, time.perf_counter()
        while True:
            call()
            reps += 1
            if time.perf_counter() - t0 >= budget_s:
                break
        sec = (time.perf_counter() - t0) / reps
        name = ("dpm (C port of the reference path)" if kind == "port"
                else "naive O(n^3)-multiply direct sum, Eq. 2 term by term (C port, exact int128)")
        return {"name": name, "value": round(nvox / sec / 1e9, 5), "unit": "GVoxel/s", "cores": threads,
                "kind": "port", "order": order, "sample": sample}
    from oracle import reference
    ref = reference.load()
    if ref is None:
        return {"name": kind, "value": None, "unit": "GVoxel/s", "cores": 1, "kind": "reference", "order": order,
                "sample": "unavailable: the reference install baseline/_ref is not on this host"}
    import importlib
    m3 = importlib.import_module("volmoments_ref.moments3d")
    harness = importlib.import_module("volmoments_ref.harness")
    rvols = [ref.Volume(np.ascontiguousarray(_as_u16(v, offset))) for v in vols]
    fn = m3.dpm_moments if kind == "ref_dpm" else m3.naive_moments

    def call():
        for rv in rvols:
            fn(rv, order)
    t0 = time.perf_counter()
    call()
    once = time.perf_counter() - t0
    reps = max(1, min(9, int(budget_s / max(once, 1e-6))))
    best, median = harness._time_best_of(call, reps, min_sample_s=0.05)
    name = "dpm_moments (reference numpy)" if kind == "ref_dpm" else "naive_moments (reference numpy)"
    return {"name": name, "value": round(nvox / best / 1e9, 5), "unit": "GVoxel/s", "cores": 1,
            "kind": "reference", "order": order, "sample": sample + f"; best of {reps} (harness._time_best_of)",
            "median_gvoxel_s": round(nvox / median / 1e9, 5)}


def cpu_baseline(cfg: int) -> dict:
    """The bounded CPU legs beside the GPU figure (~10-30 s of host work):
    the C port of the reference path (headline value), the naive direct sum,
    and the reference's own numpy dpm_moments / naive_moments."""
    legs = []
    for kind, budget in (("port", 5.0), ("naive", 3.0), ("ref_dpm", 3.0), ("ref_naive", 3.0)):
        try:
            legs.append(cpu_leg(cfg, kind, budget))
        except Exception as exc:  # reported, never fatal
            legs.append({"name": kind, "value": None, "sample": f"failed: {str(exc)[:160]}"})
    head = legs[0]
    return {"value": head.get("value"), "unit": "GVoxel/s", "cores": head.get("cores"), "kind": "port",
            "sample": head.get("sample", "") + "; exact C restatement of the reference path (oracle/)", "legs": legs}


def run_reference(args):
    """--impl reference: the CPU implementation of the reference path (the exact
    C port in oracle/, every host thread) on the SAME workload as our arm --
    the whole volume (cfg5: all 2048^3 voxels) every step -- on rank 0 only."""
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    from paper_2012_08099_b200 import configs as synth
    import oracle
    threads = os.cpu_count() or 1
    oracle.set_threads(threads)
    cfg = args.config
    order, offset = ORDER[cfg], (1024 if cfg == 3 else 0)
    if cfg == 5:
        vols = [oracle.synth_noise(2048, 2048, 0, 2048, CFG5_SEED)]
    elif cfg == 4:
        p = synth.cfg4_params(1024, 0)
        vols = [synth.cfg4_volume_numpy(p[i]) for i in range(1024)]
    else:
        vols = [{1: synth.cfg1, 2: synth.cfg2, 3: synth.cfg3}[cfg](0)] * world   # one replica per rank
    nvox = sum(int(np.prod(v.shape)) for v in vols)
    assert nvox == TOTAL_VOXELS[cfg] * (world if cfg in (1, 2, 3) else 1)

    def step():
        for v in vols:
            oracle.dpm(v, order, offset=offset)
    for _ in range(max(0, args.warmup)):
        step()
    times = []
    for _ in range(max(1, args.steps)):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
    sec = sum(times)
    value = nvox * len(times) / sec / 1e9
    sample = f"the whole workload every step ({nvox} voxels), order {order}"
    line = {
        "impl": "reference", "metric": "GVoxel/s (DPM projection -> 2D moments -> 3D moments)",
        "value": round(value, 4), "unit": "GVoxel/s", "n_gpus": world, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": round(sec / len(times) * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if cfg in (4, 5) else "weak", "vs_baseline": None, "dtype": "int64/int128 (exact)",
        "data": "synthetic (seeded; BASELINE.json configs, see paper_2012_08099_b200/configs.py)",
        "config": workload_config(cfg, world, cache_note(cfg)),
        "cpu_baseline": {"value": round(value, 4), "unit": "GVoxel/s", "cores": threads, "kind": "port",
                         "sample": sample + "; exact C restatement of the reference path (oracle/dpm_oracle.c)"},
        "e2e": {"value": round(value, 4), "unit": "GVoxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm

def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_2012_08099_b200 import _native as nat
    from paper_2012_08099_b200 import distributed as pdist
    from paper_2012_08099_b200 import configs as synth, engine

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = args.config
    order = ORDER[cfg]
    offset = 1024 if cfg == 3 else 0
    if args.simulate_ranks:
        return simulate_ranks(args, dev)

    # ---- workload: this rank's share, resident in HBM ---------------------
    z0, n_global, batch = 0, None, False
    if cfg == 5:
        L = M = N = 2048
        z0, z1 = pdist.slab_bounds(N, world, rank)
        vox = engine.synth_noise(L, M, z0, z1 - z0, CFG5_SEED, device=dev)
        n_global = N
        total_voxels = L * M * N
        scaling = "strong"
        parallelism = f"z-slab x{world}"
    elif cfg == 4:
        params = synth.cfg4_params(1024, 0)
        b0, b1 = pdist.batch_bounds(1024, world, rank)
        vox = synth.cfg4_device(params[b0:b1], device=dev)
        batch = True
        total_voxels = 1024 * 128 ** 3
        scaling = "strong"
        parallelism = f"batch x{world}"
    else:
        host = {1: synth.cfg1, 2: synth.cfg2, 3: synth.cfg3}[cfg](0)
        vox = torch.from_numpy(host).to(dev)
        total_voxels = int(np.prod(host.shape)) * world
        scaling = "weak"
        parallelism = f"replicas x{world}"
    torch.cuda.synchronize()
    my_voxels = vox.numel()
    my_bytes = my_voxels * vox.element_size()
    stream = torch.cuda.current_stream()

    # ---- one step of the hot path -------------------------------------------
    ev_p0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_p1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    launches = [0]

    graphed = stages = None
    if cfg != 5:
        graphed = engine.GraphedMoments(vox, order, offset=offset)   # captured once, replayed per step
    else:
        # three graphs with the all-reduce between; one device: the epilogue rides the moments launch
        stages = engine.GraphedSlabStages(vox, order, offset=offset, z0=z0, fused=(world == 1), n_global=n_global)

    def step(i=None):
        if cfg == 5:
            if i is not None:
                ev_p0[i].record(stream)
            stages.replay_project()
            if i is not None:
                ev_p1[i].record(stream)
            acc = stages.replay_moments2d()
            pdist.allreduce_limbs(acc)           # the z-slab exchange (no-op at N=1)
            res = stages.replay_derive()
            launches[0] += stages.launches
            return res
        res = graphed.replay()   # whole pipeline, one graph: its time is the step's (no inner events)
        launches[0] += graphed.launches
        return res

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches[0] = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l2 = int(getattr(torch.cuda.get_device_properties(dev), "L2_cache_size", 126 << 20) or (126 << 20))
    flush_l2 = my_bytes <= l2
    with ClockSampler(local) as clk:
        if flush_l2:
            # input fits in L2: scrub L2 (untimed write of 2x its size) before
            # every step and time each step with its own event pair
            scrub = torch.empty(2 * l2 // 4, dtype=torch.int32, device=dev)
            es = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            ee = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
            for i in range(args.steps):
                scrub.fill_(i)
                es[i].record(stream)
                res = step(i)
                ee[i].record(stream)
            torch.cuda.synchronize()
        else:
            e0.record(stream)
            for i in range(args.steps):
                res = step(i)
            e1.record(stream)
            torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in zip(es, ee)) if flush_l2 else e0.elapsed_time(e1)
    # cfg5: the projection stage between its own events; other configs: the
    # roofline kernel is the whole graph replay, i.e. the step itself
    proj_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev_p0, ev_p1)) if cfg == 5 else ms / args.steps
    st = res.status.cpu()
    if int(st.max().item()) != 0:
        raise RuntimeError(f"device consistency status {st.tolist()}")
    t = torch.tensor([ms, proj_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, proj_max = float(t[0]), float(t[1])
    value = total_voxels * args.steps / (ms_max * 1e-3) / 1e9

    # ---- e2e through the public API -----------------------------------------
    e2e = e2e_pinned = None
    if not args.no_e2e:
        e2e_pinned = run_e2e(args, cfg, order, offset, vox, z0, n_global, world, rank, dev, total_voxels)
        e2e = run_e2e_dropin(args, cfg, order, offset, vox) if world == 1 else e2e_pinned

    # ---- CPU baseline (rank 0, N=1 only) -------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg)

    peak, peak_kind = measured_peak_gbs()
    achieved = my_bytes / (proj_max * 1e-3) / 1e9
    key = f"cfg{cfg}_n{world}"
    tr = ncu_traffic(key)
    line = {
        "metric": "GVoxel/s (DPM projection -> 2D moments -> 3D moments)",
        "value": round(value, 2), "unit": "GVoxel/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "u16" if vox.element_size() == 2 else "u8",
        "data": "synthetic (seeded; BASELINE.json configs, see paper_2012_08099_b200/configs.py)",
        "config": workload_config(cfg, world, cache_note(cfg)),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     # the same bytes over the WHOLE step (zeroing, moments and epilogue launches included)
                     "frac_step": round(my_bytes / (ms_max / args.steps * 1e-3) / 1e9 / peak, 4),
                     "kernel": "zstream_kernel (the layout-T projection pass alone; its buffers are re-zeroed by the moments stage)" if cfg == 5 else "whole pipeline (one graph replay)",
                     "traffic": tr},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "e2e_pinned": e2e_pinned,
        "gpu_launches": launches[0],
        "clocks": clk.summary(),
        "stage_ms": {"projection": round(proj_max, 4), "step": round(ms_max / args.steps, 4)},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def simulate_ranks(args, dev):
    """--simulate-ranks G (cfg5): the per-rank step of a G-way z-slab split,
    timed on this single GPU one rank at a time -- the rank's 2048/G planes at
    their global z0 (generated on the device), projection + exact 2D moments in
    global coordinates + epilogue as separate stages (``fused=False``: at N > 1
    the all-reduce sits between them).  Predicts the G-GPU figure as
    total voxels / (slowest rank's step + an assumed all-reduce latency); the
    multi-GPU run itself is not measured here (one GPU)."""
    import torch

    from paper_2012_08099_b200 import distributed as pdist
    from paper_2012_08099_b200 import engine
    if args.config != 5:
        raise SystemExit("--simulate-ranks applies to the z-slab config (--config 5)")
    G = args.simulate_ranks
    L = M = N = 2048
    allreduce_us = 25.0   # assumption: one NCCL all-reduce of 2.7 KiB over NVLink (latency-bound)
    stream = torch.cuda.current_stream()

    def time_split(g):
        per = []
        for r in range(g):
            z0, z1 = pdist.slab_bounds(N, g, r)
            slab = engine.synth_noise(L, M, z0, z1 - z0, CFG5_SEED, device=dev)
            st = engine.GraphedSlabStages(slab, 6, z0=z0, fused=False, n_global=N)
            for _ in range(max(3, args.warmup)):
                st.replay_project(); st.replay_moments2d(); st.replay_derive()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(args.steps):
                st.replay_project(); st.replay_moments2d(); res = st.replay_derive()
            e1.record(stream)
            torch.cuda.synchronize()
            assert int(res.status[0]) == 0
            per.append(e0.elapsed_time(e1) / args.steps)
            del st, slab
            torch.cuda.empty_cache()
        return per
    one = time_split(1)[0]
    per = time_split(G)
    t_pred = max(per) + allreduce_us * 1e-3
    value = L * M * N / (t_pred * 1e-3) / 1e9
    line = {"metric": "GVoxel/s (DPM projection -> 2D moments -> 3D moments)", "simulated_gpus": G,
            "unit": "GVoxel/s", "steps": args.steps, "config": workload_config(5, G, cache_note(5)),
            "per_rank_ms": [round(t, 4) for t in per], "n1_unfused_ms": round(one, 4),
            "assumed_allreduce_us": allreduce_us, "predicted_ms_per_step": round(t_pred, 4),
            "predicted_value": round(value, 1), "n1_value": round(L * M * N / (one * 1e-3) / 1e9, 1),
            "predicted_efficiency": round(one / (G * t_pred), 4),
            "note": "per-rank steps timed one at a time on ONE GPU; the multi-GPU run is not measured"}
    print(json.dumps(line), flush=True)
    return 0


def run_e2e_dropin(args, cfg, order, offset, vox):
    """The drop-in call of the reference API on HOST numpy data, every step:
    ``dpm_moments(Volume(voxels), order)`` (moments3d.py:232-264 signature;
    ``dpm_moments_batch`` for the cfg4 batch) -- pageable host memory -> the
    package's threaded pinned-staging upload -> the device pipeline -> exact
    Python ints.  cfg3's int16 CT volume is offset to uint16 on the host first
    (untimed), as the reference's callers must (its Volume is uint8/uint16 only)."""
    import torch

    import paper_2012_08099_b200 as vm
    try:
        host = vox.cpu().numpy()
        if cfg == 3:
            host = (host.astype(np.int32) + offset).astype(np.uint16)
        if cfg == 4:
            def call():
                return vm.dpm_moments_batch(host, order)
            path = "paper_2012_08099_b200.dpm_moments_batch(numpy [1024,128,128,128] uint8, 3) -> exact ints"
        else:
            volume = vm.Volume(host)

            def call():
                return vm.dpm_moments(volume, order)
            path = f"paper_2012_08099_b200.dpm_moments(Volume(numpy {host.dtype}), {order}) -> exact ints"
        call()
        call()
        torch.cuda.synchronize()
        steps = max(1, min(args.steps, 3)) if host.nbytes > (1 << 30) else max(1, args.steps)
        t0 = time.perf_counter()
        for _ in range(steps):
            res = call()
        sec = time.perf_counter() - t0
        n3d = len(vm.moment_indices(order))
        nvol = len(res) if isinstance(res, list) else 1
        return {"value": round(host.size * steps / sec / 1e9, 3), "unit": "GVoxel/s",
                "h2d_bytes_per_step": int(host.nbytes), "d2h_bytes_per_step": int(nvol * (n3d * 16 + 4)),
                "steps": steps, "path": path + " (pageable host memory, wall clock)"}
    except Exception as exc:
        return {"value": None, "unit": "GVoxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "error": str(exc)[:200]}


def run_e2e(args, cfg, order, offset, vox, z0, n_global, world, rank, dev, total_voxels):
    """Same metric through the host-buffer API, every step: pinned host volume
    -> device -> moments -> exact result back in host memory.  Volumes that fit
    in one piece replay one CUDA graph (engine.HostGraphedMoments); the z-slab
    config streams 64-plane chunks with H2D overlapped with the pass
    (streaming.HostStreamer)."""
    import torch
    import torch.distributed as dist

    from paper_2012_08099_b200 import distributed as pdist
    from paper_2012_08099_b200 import engine
    from paper_2012_08099_b200.streaming import HostStreamer
    try:
        host = torch.empty(tuple(vox.shape), dtype=vox.dtype, pin_memory=True)
        host.copy_(vox)
        h2d = host.numel() * host.element_size()
        zslab = cfg == 5   # z-slab sharded: 2D-moment limbs are all-reduced before the epilogue
        if not zslab and h2d <= (4 << 30):
            # fits on the device in one piece: H2D + pipeline + D2H captured in one CUDA graph
            hg = engine.HostGraphedMoments(host, order, offset=offset, device=dev)
            path = "paper_2012_08099_b200.engine.HostGraphedMoments (pinned host, one graph: H2D, projection + moments/epilogue kernels, D2H)"

            def step():
                return hg.run()
        else:
            streamer = HostStreamer(tuple(vox.shape), vox.dtype, order, chunk_planes=64, device=dev)
            path = "paper_2012_08099_b200.streaming.HostStreamer (pinned host, 64-plane chunks)"

            def step():
                acc = streamer.run(host, offset=offset, z_base=z0, n_global=n_global)
                pdist.allreduce_limbs(acc)
                res = engine.derive(acc, order, kind=engine.acc_kind(vox, order))
                return res.i128.to("cpu", non_blocking=False), res.status.to("cpu", non_blocking=False)
        torch.cuda.synchronize()

        for _ in range(2):
            step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        steps = max(1, min(args.steps, 3)) if h2d > (1 << 30) else max(1, args.steps)
        for _ in range(steps):
            out, st = step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        wall = (time.perf_counter() - t0) * 1e3
        t = torch.tensor([max(ms, wall)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        d2h = out.numel() * out.element_size() + st.numel() * st.element_size()
        return {"value": round(total_voxels * steps / (float(t[0]) * 1e-3) / 1e9, 3), "unit": "GVoxel/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps,
                "path": path}
    except Exception as exc:
        return {"value": None, "unit": "GVoxel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "error": str(exc)[:200]}


if __name__ == "__main__":
    sys.exit(main())
