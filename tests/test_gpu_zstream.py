"""Layout T: the moments pipeline of wide volumes builds the
method's images of the volume with x and z exchanged, with the z-streaming
kernel (csrc/project_zstream.cu).  Its images must equal the reference-layout
images of the transposed volume bit for bit (through ``project``, an
independent kernel), its profile a numpy restatement, and its moments the
oracle -- for every order, dtype, partial tile and schedule."""
import numpy as np
import pytest
import torch

import oracle
import paper_2012_08099_b200 as vm
from paper_2012_08099_b200 import engine

pytestmark = pytest.mark.gpu


def np_profile(vol: np.ndarray, t: int) -> np.ndarray:
    n, m, l = vol.shape
    at = abs(t)
    out = np.zeros(l + at * (n - 1), dtype=np.int64)
    cols = vol.astype(np.int64).sum(axis=1)
    x = np.arange(l)
    for z in range(n):
        np.add.at(out, x + t * z + (at * (n - 1) if t < 0 else 0), cols[z])
    return out


def _vol(shape, dt, seed):
    rng = np.random.default_rng(seed)
    if dt == np.int16:
        return rng.integers(-1024, 3072, size=shape).astype(np.int16)
    return rng.integers(0, np.iinfo(dt).max + 1, size=shape).astype(dt)


SHAPES = [
    ((16, 12, 256), np.uint16),     # one y-group, two steps
    ((37, 25, 264), np.uint16),     # partial x-tile, partial y-group, partial last z-step
    ((9, 30, 512), np.uint16),      # two x-tiles, two steps (second partial)
    ((130, 13, 256), np.uint8),     # uint8 8-wide lanes, many steps
    ((21, 7, 200), np.int16),       # int16 + offset, partial everything
    ((300, 20, 256), np.uint16),    # long columns: ring slots wrap many times
]


@pytest.mark.parametrize("order", [3, 4, 5, 6])
@pytest.mark.parametrize("shape,dt", SHAPES)
def test_layout_t_images_and_profile(order, shape, dt):
    vol = _vol(shape, dt, sum(shape) + order)
    off = 1024 if dt == np.int16 else 0
    v = torch.from_numpy(vol).cuda()
    assert engine.acc_kind(v, order, off) == "profile_t"
    imgs, prof = engine.project_profile(v, order, offset=off)
    src = vol.astype(np.int32) + off if off else vol
    src_t = np.ascontiguousarray(src.transpose(2, 1, 0)).astype(np.uint16 if dt != np.uint8 else np.uint8)
    want = oracle.project(src_t, engine.num_images(order))
    torch.cuda.synchronize()
    for k in range(engine.num_images(order)):
        if k == 2:
            continue
        got = imgs[k][0].cpu().numpy().view(np.uint32).astype(np.int64)
        assert np.array_equal(got, want[k]), k
    t = {3: -1, 4: 2, 5: -2, 6: 3}[order]
    assert np.array_equal(prof[0].cpu().numpy(), np_profile(src_t.astype(np.int64), t))


@pytest.mark.parametrize("order", [3, 4, 5, 6])
@pytest.mark.parametrize("shape,dt", SHAPES)
def test_layout_t_moments_match_oracle(order, shape, dt):
    vol = _vol(shape, dt, 3 * sum(shape) + order)
    if dt == np.int16:
        res = engine.moments(torch.from_numpy(vol).cuda(), order, offset=1024)
        torch.cuda.synchronize()
        assert int(res.status[0]) == 0
        want = oracle.naive((vol.astype(np.int32) + 1024).astype(np.uint16), order)
        assert engine.i128_to_ints(res.i128[0].cpu().numpy()) == [want[k] for k in vm.moment_indices(order)]
    else:
        assert vm.dpm_moments(vm.Volume(vol), order).values == oracle.naive(vol, order)


@pytest.mark.parametrize("order", [4, 6])
def test_layout_t_zslabs_compose(order):
    vol = _vol((90, 14, 264), np.uint16, order)
    whole = vm.dpm_moments(vm.Volume(vol), order).values
    for cuts in ([0, 45, 90], [0, 1, 9, 50, 90]):
        acc = None
        for z0, z1 in zip(cuts[:-1], cuts[1:]):
            part = engine.moments2d_partial(torch.from_numpy(vol[z0:z1]).cuda(), order, z0=z0)
            acc = part.clone() if acc is None else acc + part
        res = engine.derive(acc, order, kind="profile_t")
        torch.cuda.synchronize()
        assert int(res.status[0]) == 0
        assert dict(zip(vm.moment_indices(order), engine.i128_to_ints(res.i128[0].cpu().numpy()))) == whole


def test_layout_t_batch():
    vols = np.stack([_vol((20, 13, 256), np.uint16, s) for s in range(3)])
    got = vm.dpm_moments_batch(vols, 6)
    for b in range(3):
        assert got[b].values == oracle.naive(vols[b], 6)


def test_layout_t_unreadable_rows_use_the_transposed_generic_kernel():
    """A batch (no staged pass) with L >= 192 but L % 8 != 0, which the TMA
    kernel cannot read: the generic brick kernel builds the same layout-T
    images on the transposed view."""
    base = np.stack([_vol((20, 9, 208), np.uint16, s) for s in (7, 8)])
    v = torch.from_numpy(base).cuda()[:, :, :, :203]       # row pitch 208, width 203
    res = engine.moments(v, 5)
    torch.cuda.synchronize()
    for b in range(2):
        want = oracle.naive(np.ascontiguousarray(base[b, :, :, :203]), 5)
        assert engine.i128_to_ints(res.i128[b].cpu().numpy()) == [want[k] for k in vm.moment_indices(5)]


def test_layout_t_full_size_slab_schedule():
    """A 2048-wide slab large enough for the round-robin z-split schedule."""
    vol = engine.synth_noise(2048, 256, 0, 128, 9)
    res = engine.moments(vol, 6)
    torch.cuda.synchronize()
    assert int(res.status[0]) == 0
    oracle.set_threads(oracle.max_threads())
    want = oracle.dpm(vol.cpu().numpy(), 6)
    assert dict(zip(vm.moment_indices(6), engine.i128_to_ints(res.i128[0].cpu().numpy()))) == want


@pytest.mark.parametrize("order", [3, 4, 5, 6])
@pytest.mark.parametrize("offset,lo,hi", [(1024, -1024, 3071), (32768, -32768, 32767), (40000, -32768, 25535),
                                          (1, -1, 5000)])
def test_signed_exact_int16(order, offset, lo, hi):
    """Signed-exact int16 (dpm_moments on layout-T volumes): the pass sums the raw
    signed voxels (no per-voxel offset add) and the epilogue adds offset x the
    box's moments; exact against the oracle on the offset uint16 volume, for
    the extreme ends of the range, a batch, ragged shapes."""
    rng = np.random.default_rng(order * 7 + offset % 97)
    vols = rng.integers(lo, hi + 1, size=(3, 21, 13, 200), dtype=np.int64).astype(np.int16)
    vols[0, :2] = lo                                   # both ends of the allowed range in one volume
    vols[0, -2:] = hi
    res = engine.moments(torch.from_numpy(vols).cuda(), order, offset=offset)
    torch.cuda.synchronize()
    assert res.status.cpu().numpy().max() == 0
    idx = vm.moment_indices(order)
    for b in range(3):
        want = oracle.naive((vols[b].astype(np.int32) + offset).astype(np.uint16), order)
        assert engine.i128_to_ints(res.i128[b].cpu().numpy()) == [want[k] for k in idx], b
        assert np.isclose(res.f64[b].cpu().numpy()[0], float(want[(0, 0, 0)]))


@pytest.mark.parametrize("yb", [2, 4, 100])
def test_blocked_column_order(yb):
    """Large image sets order the columns in blocks of y-groups with the x-tile
    outermost inside a block (project_zstream.cu, zdecode).  DPM_ZS_XT_MAJOR_MB=0
    selects that order for small volumes in a fresh process and DPM_ZS_YB sets
    the block size (2, 4: short last blocks; 100: one block = plain x-tile
    outermost): orders 4 and 6, three x-tiles, partial tiles, and a batch of
    three volumes at order 5, vs the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import numpy as np, torch, oracle\n"
        "import paper_2012_08099_b200 as vm\n"
        "from paper_2012_08099_b200 import engine\n"
        "rng = np.random.default_rng(77)\n"
        "for shape, order in (((40, 50, 712), 6), ((24, 37, 520), 4)):\n"
        "    vol = rng.integers(0, 65536, size=shape).astype(np.uint16)\n"
        "    res = engine.moments(torch.from_numpy(vol).cuda(), order)\n"
        "    torch.cuda.synchronize()\n"
        "    assert int(res.status[0]) == 0\n"
        "    want = oracle.dpm(vol, order)\n"
        "    got = engine.i128_to_ints(res.i128[0].cpu().numpy())\n"
        "    assert got == [want[k] for k in vm.moment_indices(order)], (shape, order)\n"
        "vols = rng.integers(0, 65536, size=(3, 16, 40, 520)).astype(np.uint16)\n"
        "res = engine.moments(torch.from_numpy(vols).cuda(), 5)\n"
        "torch.cuda.synchronize()\n"
        "for b in range(3):\n"
        "    want = oracle.dpm(vols[b], 5)\n"
        "    assert int(res.status[b]) == 0\n"
        "    assert engine.i128_to_ints(res.i128[b].cpu().numpy()) == [want[k] for k in vm.moment_indices(5)], b\n"
        "print('blocked order ok')\n")
    env = dict(os.environ, DPM_ZS_XT_MAJOR_MB="0", DPM_ZS_YB=str(yb), PYTHONPATH=root)
    proc = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, cwd=root, timeout=600)
    assert proc.returncode == 0 and "blocked order ok" in proc.stdout, proc.stdout + proc.stderr
