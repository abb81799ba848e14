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
