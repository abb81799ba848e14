"""Multi-rank host logic on CPU (gloo, world_size 2): z-slab partition, exact
limb all-reduce, batch partition.  The per-rank compute is the oracle's
2D-moment step in global coordinates (the device path is covered by -m gpu)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2012_08099_b200 import distributed as pdist
from paper_2012_08099_b200 import engine


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, vol, order, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = vol.shape[0]
        z0, z1 = pdist.slab_bounds(n, world, rank)
        slab = np.ascontiguousarray(vol[z0:z1])
        dims = (vol.shape[2], vol.shape[1], z1 - z0)
        blocks = []
        imgs = oracle.project(slab, oracle.num_images(order)) if z1 > z0 else None
        for k in range(oracle.num_images(order)):
            if imgs is None:
                m = {pq: 0 for pq in oracle.moments2d(np.zeros((1, 1), np.int64), order)}
            else:
                W, H, ai, aj = oracle.layout(dims, k, z0)
                m = oracle.moments2d(imgs[k], order, ai, aj)
            blocks.append([m[pq] for pq in sorted(m, key=lambda t: (t[0], t[1]))])
        acc = torch.from_numpy(engine.ints_to_limbs(blocks)[None])
        pdist.allreduce_limbs(acc)
        total = engine.acc_to_ints(acc.numpy())[0]
        keys = sorted(oracle.moments2d(np.zeros((1, 1), np.int64), order), key=lambda t: (t[0], t[1]))
        m2d = [dict(zip(keys, row)) for row in total]
        vals, st = oracle.derive3d(m2d, order)
        q.put((rank, st, vals))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("order", [4, 6])
def test_zslab_allreduce_world2_matches_whole_volume(order):
    vol = np.random.default_rng(order).integers(0, 65536, (13, 6, 9), dtype=np.uint16)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, vol, order, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(60)
    want = oracle.dpm(vol, order)
    for rank, st, vals in out:
        assert st == 0 and vals == want, rank


def test_slab_and_batch_bounds_cover_exactly():
    for n in (1, 2, 7, 2048, 2049):
        for world in (1, 2, 3, 4, 8):
            spans = [pdist.slab_bounds(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    assert pdist.batch_bounds(1024, 8, 3) == (384, 512)
    with pytest.raises(ValueError):
        pdist.slab_bounds(10, 2, 2)


def _gather_worker(rank, world, port, counts, q):
    """moments_batch_sharded(gather=True) with a CPU stand-in for the device
    engine (engine.moments replaced by the oracle): uneven shards are padded,
    all-gathered and trimmed back in rank order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2012_08099_b200.engine import DeviceMoments
        rng = np.random.default_rng(100)
        vols = rng.integers(0, 256, (sum(counts), 5, 4, 6), dtype=np.uint8)
        b0 = sum(counts[:rank])
        mine = torch.from_numpy(vols[b0:b0 + counts[rank]])

        def cpu_moments(v, order, offset=0, **_):
            rows = [[float(x) for x in oracle.dpm(v[b].numpy(), order).values()] for b in range(v.shape[0])]
            f64 = torch.tensor(rows, dtype=torch.float64).reshape(v.shape[0], -1)
            return DeviceMoments(i128=None, f64=f64, status=torch.zeros(v.shape[0], dtype=torch.int32), launches=0)
        engine.moments = cpu_moments
        res, gathered = pdist.moments_batch_sharded(mine, 3, gather=True)
        q.put((rank, gathered.numpy().tolist()))
    finally:
        dist.destroy_process_group()


def test_batch_sharded_gather_world2():
    counts = [3, 2]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 2, port, counts, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
    rng = np.random.default_rng(100)
    vols = rng.integers(0, 256, (5, 5, 4, 6), dtype=np.uint8)
    want = [[float(x) for x in oracle.dpm(vols[b], 3).values()] for b in range(5)]
    assert out[0] == want and out[1] == want


def _fused_guard_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        try:
            engine.GraphedSlabStages(torch.zeros((8, 4, 256), dtype=torch.uint16), 4, fused=True)
            q.put((rank, "no error"))
        except ValueError as exc:
            q.put((rank, "ValueError" if "fused" in str(exc) else str(exc)))
    finally:
        dist.destroy_process_group()


def test_fused_slab_stages_refused_in_a_multirank_group():
    """fused=True would run the epilogue before the limb all-reduce."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_fused_guard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(60)
    assert out == {0: "ValueError", 1: "ValueError"}
