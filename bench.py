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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
# reference arm: the CPU port of the reference path (oracle/, C + OpenMP)

def cpu_sample_cfg(cfg: int):
    """A bounded sample of the workload for the CPU leg: (voxels, order, offset, description)."""
    from paper_2012_08099_b200 import configs as synth
    if cfg == 5:
        import oracle
        planes = 32
        v = oracle.synth_noise(2048, 2048, 0, planes, CFG5_SEED)
        return v, 6, 0, f"first {planes} planes of the cfg5 volume (2048x2048x{planes}), order 6"
    if cfg == 4:
        p = synth.cfg4_params(16, 0)
        v = np.stack([synth.cfg4_volume_numpy(p[i]) for i in range(16)])
        return v, 3, 0, "16 of the 1024 cfg4 volumes, order 3"
    if cfg == 3:
        return synth.cfg3(0), 4, 1024, "the whole cfg3 volume, order 4"
    if cfg == 2:
        return synth.cfg2(0), 3, 0, "the whole cfg2 volume, order 3"
    return synth.cfg1(0), 3, 0, "the whole cfg1 volume, order 3"


def time_cpu(v, order, offset, min_seconds=8.0, max_reps=50):
    import oracle
    reps, t0 = 0, time.perf_counter()
    while True:
        if v.ndim == 4:
            for b in range(v.shape[0]):
                oracle.dpm(v[b], order, offset=offset)
        else:
            oracle.dpm(v, order, offset=offset)
        reps += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or reps >= max_reps:
            return el / reps


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    import oracle
    threads = os.cpu_count() or 1
    oracle.set_threads(threads)
    v, order, offset, sample = cpu_sample_cfg(args.config)
    nvox = int(np.prod(v.shape))
    for _ in range(max(0, args.warmup)):
        time_cpu(v, order, offset, min_seconds=0.0, max_reps=1)
    times = [time_cpu(v, order, offset, min_seconds=0.0, max_reps=1) for _ in range(max(1, args.steps))]
    sec = sum(times)
    value = nvox * len(times) / sec / 1e9
    line = {
        "impl": "reference", "metric": "GVoxel/s (DPM projection -> 2D moments -> 3D moments)",
        "value": round(value, 4), "unit": "GVoxel/s", "n_gpus": world, "steps": len(times), "warmup": args.warmup,
        "ms_per_step": round(sec / len(times) * 1e3, 3), "higher_is_better": True, "scaling": "replicas only",
        "vs_baseline": None, "dtype": "int64/int128 (exact)", "data": "synthetic (seeded)",
        "config": {"workload": CONFIG_DESC[args.config], "order": order},
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
    order = {1: 3, 2: 3, 3: 4, 4: 3, 5: 6}[cfg]
    offset = 1024 if cfg == 3 else 0

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
        stages = engine.GraphedSlabStages(vox, order, offset=offset, z0=z0, fused=(world == 1))

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
        if i is not None:
            ev_p0[i].record(stream)
        res = graphed.replay()
        if i is not None:
            ev_p1[i].record(stream)   # whole pipeline (projection dominates)
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
    proj_ms = statistics.mean(a.elapsed_time(b) for a, b in zip(ev_p0, ev_p1))
    st = res.status.cpu()
    if int(st.max().item()) != 0:
        raise RuntimeError(f"device consistency status {st.tolist()}")
    t = torch.tensor([ms, proj_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max, proj_max = float(t[0]), float(t[1])
    value = total_voxels * args.steps / (ms_max * 1e-3) / 1e9

    # ---- e2e through the host-buffer API ------------------------------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, cfg, order, offset, vox, z0, n_global, world, rank, dev, total_voxels)

    # ---- CPU baseline (rank 0, N=1 only) -------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            threads = os.cpu_count() or 1
            oracle.set_threads(threads)
            v, o, off, sample = cpu_sample_cfg(cfg)
            sec = time_cpu(v, o, off, min_seconds=8.0)
            cpu = {"value": round(int(np.prod(v.shape)) / sec / 1e9, 4), "unit": "GVoxel/s", "cores": threads,
                   "kind": "port", "sample": sample + "; exact C restatement of the reference path (oracle/)"}
        except Exception as exc:  # reported, never fatal
            cpu = {"value": None, "unit": "GVoxel/s", "cores": None, "kind": "port", "sample": f"failed: {exc}"}

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
        "config": {"workload": CONFIG_DESC[cfg], "order": order, "parallelism": parallelism,
                   "voxels_per_step": total_voxels, "cache": "L2 scrubbed before every step (untimed 2xL2 write), per-step events"
                   if flush_l2 else "inputs larger than L2 (no flush)"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "peak_kind": peak_kind,
                     "kernel": "project_stream (projection stage incl. image zeroing)" if cfg == 5 else "whole pipeline",
                     "traffic": tr},
        "cpu_baseline": cpu,
        "e2e": e2e,
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
