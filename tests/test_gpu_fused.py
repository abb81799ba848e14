"""The one-launch moments pass of small uint8 volumes (csrc/project_fused.cu:
order 3, x and z extents <= 128, any height): packed-byte folds, row-by-row
y-power accumulators, per-volume reduction and the epilogue of the last CTA.
Every case is compared with the oracle (oracle/dpm_oracle.c, pinned to the
reference's golden outputs) and must run as one pass after the zeroing kernel
(programmatic dependent launch: the pass starts while the zeroing drains)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2012_08099_b200 as vm
from paper_2012_08099_b200 import engine

pytestmark = pytest.mark.gpu

IDX3 = vm.moment_indices(3)


def _check(vol: np.ndarray, launches: int | None = 2):
    """vol: one (N, M, L) or a batch (B, N, M, L) of uint8 volumes (rows of
    16-byte multiples: the TMA reads them in place)."""
    dev = torch.from_numpy(vol).cuda()
    res = engine.moments(dev, 3)
    torch.cuda.synchronize()
    if launches is not None:
        assert res.launches == launches
    assert int(res.status.max()) == 0
    got = res.i128.cpu().numpy()
    vols = vol if vol.ndim == 4 else vol[None]
    for b in range(vols.shape[0]):
        want = oracle.dpm(np.ascontiguousarray(vols[b]), 3)
        assert engine.i128_to_ints(got[b]) == [want[k] for k in IDX3], f"volume {b}"
    f64 = res.f64.cpu().numpy()
    assert np.array_equal(f64[:, 0], vols.reshape(vols.shape[0], -1).sum(axis=1).astype(np.float64))


@pytest.mark.parametrize("shape", [
    (64, 64, 64),        # config 1
    (128, 128, 128),     # a config-4 volume alone
    (1, 1, 16),          # one plane, one row
    (7, 3, 48),          # ragged z, y, partial warps and lanes
    (128, 300, 128),     # > 128 rows: the packed profile window is flushed mid-volume
    (100, 1024, 112),    # the tallest volume the kernel takes
    (33, 17, 128),
])
def test_fused_single_volume_max_values(shape):
    rng = np.random.default_rng(sum(shape))
    vol = rng.integers(0, 256, size=shape, dtype=np.uint8)
    vol[..., :2] = 255            # saturated corners: the 16-bit fields at their bounds
    vol[:2] = 255
    _check(vol)


def test_fused_all_255():
    _check(np.full((128, 128, 128), 255, dtype=np.uint8))


@pytest.mark.parametrize("B,shape,seed", [(37, (24, 40, 64), 1), (300, (16, 9, 16), 2), (5, (128, 128, 128), 3)])
def test_fused_batch_runs_split_volumes(B, shape, seed):
    # more row-steps than CTAs and volumes split between CTAs at arbitrary rows:
    # partial-volume reductions and the per-volume completion counter
    rng = np.random.default_rng(seed)
    vol = rng.integers(0, 256, size=(B,) + shape, dtype=np.uint8)
    _check(vol)


def test_fused_binary_batch_like_config4():
    from paper_2012_08099_b200 import configs as synth
    params = synth.cfg4_params(24, 0)
    dev = synth.cfg4_device(params)
    res = engine.moments(dev, 3)
    torch.cuda.synchronize()
    assert res.launches == 2   # the accumulator zeroing kernel + the fused pass
    host = dev.cpu().numpy()
    got = res.i128.cpu().numpy()
    for b in range(24):
        want = oracle.dpm(host[b], 3)
        assert engine.i128_to_ints(got[b]) == [want[k] for k in IDX3], b


def test_fused_graph_replays_are_identical():
    rng = np.random.default_rng(9)
    vol = torch.from_numpy(rng.integers(0, 256, size=(11, 128, 64, 128), dtype=np.uint8)).cuda()
    g = engine.GraphedMoments(vol, 3)
    first = g.replay().i128.clone()
    for _ in range(3):
        again = g.replay().i128
    torch.cuda.synchronize()
    assert torch.equal(first, again)
    host = vol.cpu().numpy()
    for b in (0, 10):
        want = oracle.dpm(host[b], 3)
        assert engine.i128_to_ints(first[b].cpu().numpy()) == [want[k] for k in IDX3]


def test_not_fused_outside_envelope():
    # order 4, uint16, wider than 128 or deeper than 128: the streaming pipeline (> 1 launch)
    rng = np.random.default_rng(4)
    for vol, order in ((rng.integers(0, 256, (16, 8, 64), dtype=np.uint8), 4),
                       (rng.integers(0, 256, (130, 8, 64), dtype=np.uint8), 3),
                       (rng.integers(0, 4096, (16, 8, 64), dtype=np.uint16), 3)):
        res = engine.moments(torch.from_numpy(vol).cuda(), order)
        torch.cuda.synchronize()
        assert res.launches >= 3   # zeroing, projection, moments (+ epilogue)
        want = oracle.dpm(vol, order)
        assert engine.i128_to_ints(res.i128[0].cpu().numpy()) == [want[k] for k in vm.moment_indices(order)]


def test_dropin_batch_from_host_numpy():
    """dpm_moments_batch on a host numpy batch above the staging threshold: the
    threaded pinned-staging upload (volumes along the leading axis), then the
    fused pass; exact against the oracle."""
    rng = np.random.default_rng(21)
    vols = rng.integers(0, 256, size=(40, 128, 64, 128), dtype=np.uint8)   # 40 MB
    got = vm.dpm_moments_batch(vols, 3)
    for b in (0, 17, 39):
        assert got[b].values == oracle.dpm(vols[b], 3), b
