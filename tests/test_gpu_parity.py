"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
outputs (tests/golden/, generated from /root/reference) and the C oracle.

Projections are bit-exact; moments are exact integers (the reference returns
exact Python ints; our fp64 copies are therefore within 1 ulp)."""
import numpy as np
import pytest
import torch

import oracle
import pyoracle
import paper_2012_08099_b200 as vm
from golden_data import (ORIENTATIONS, configs, moments, parse_moments, projections, sha,
                         volume_for)
from paper_2012_08099_b200 import _native as nat, configs as synth, engine
from paper_2012_08099_b200.errors import InconsistencyError

pytestmark = pytest.mark.gpu


def _ints(res, b=0):
    return engine.i128_to_ints(res.i128[b].cpu().numpy())


def test_golden_projections_bit_exact(cuda):
    vols, imgs = projections()
    for name, v in vols.items():
        ps = vm.project_all(vm.Volume(v.copy()))
        for o in vm.Orientation:
            assert np.array_equal(ps[o].pixels, imgs[(name, o.value)]), (name, o)
        assert ps.anti.origin_offset == v.shape[0] - 1


@pytest.mark.parametrize("K", [3, 4])
def test_golden_moments_exact(cuda, K):
    for name, entry in moments().items():
        v = volume_for(name)
        got = vm.dpm_moments(vm.Volume(v.copy()), K)
        assert got.values == parse_moments(entry[f"dpm{K}"]), name


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4_0", "cfg4_1", "cfg4_2", "cfg4_3", "cfg5_slab"])
def test_golden_configs(cuda, name):
    c = configs()[name]
    p = c["params"]
    off = p.get("offset", 0)
    if name == "cfg1":
        v = synth.cfg1(p["seed"])
    elif name == "cfg2":
        v = synth.cfg2(p["seed"])
    elif name == "cfg3":
        v = synth.cfg3(p["seed"])
    elif name.startswith("cfg4"):
        v = synth.cfg4_volume_numpy(synth.cfg4_params(4, p["seed"])[p["index"]])
    else:
        v = engine.synth_noise(p["L"], p["M"], p["z0"], p["nz"], p["seed"]).cpu().numpy()
    assert sha(v) == c["voxels_sha256"]
    t = torch.from_numpy(v).cuda()
    res = engine.moments(t, c["order"], offset=off)
    torch.cuda.synchronize()
    assert int(res.status[0]) == 0
    want = parse_moments(c["dpm"])
    assert dict(zip(vm.moment_indices(c["order"]), _ints(res))) == want
    f64 = res.f64[0].cpu().numpy()
    exact = np.array([float(want[k]) for k in vm.moment_indices(c["order"])])
    assert np.all(np.abs(f64 - exact) <= 1e-12 * np.maximum(np.abs(exact), 1.0))
    imgs = engine.project(t, 5, offset=off)
    torch.cuda.synchronize()
    for k, o in enumerate(ORIENTATIONS):
        px = imgs[k][0].cpu().numpy().view(np.uint32).astype(np.int64)
        assert sha(px) == c["images_sha256"][o], o


@pytest.mark.parametrize("K", [5, 6])
def test_orders_5_6_against_loop_oracle(cuda, K):
    for seed, dims in enumerate([(5, 4, 3), (2, 6, 5), (7, 1, 4), (1, 1, 1)]):
        v = vm.random(dims, 16, seed=seed)
        assert vm.dpm_moments(v, K).values == pyoracle.moments_3d(v.voxels, K)


def test_known_answers(cuda):
    v = vm.delta((4, 5, 6), (1, 2, 3), 5)                      # test_moments3d.py:25-30
    for K in (3, 4, 5, 6):
        for (p, q, r), val in vm.dpm_moments(v, K).items():
            assert val == 5 * 1 ** p * 2 ** q * 3 ** r
    t = vm.dpm_moments(vm.uniform((2, 2, 2), 1), 4)          # :33-40
    assert (t.mass, t[(1, 0, 0)], t[(1, 1, 0)], t[(1, 1, 1)]) == (8, 4, 2, 1)
    g = np.zeros((4, 4, 4), np.uint8); g[0, 0, 0] = 1; g[3, 2, 1] = 2    # :43-51
    t = vm.dpm_moments(vm.Volume(g), 4)
    assert (t[(1, 1, 1)], t[(2, 1, 1)], t[(1, 2, 1)]) == (12, 12, 24)
    img = vm.project(vm.delta((4, 4, 4), (1, 0, 1), 7), vm.Orientation.DIAG)   # test_projection.py:44-49
    assert np.argwhere(img.pixels).tolist() == [[0, 2]] and img.pixels[0, 2] == 7
    img = vm.project(vm.delta((4, 4, 4), (0, 2, 3), 7), vm.Orientation.ANTI)   # :52-56
    assert img.origin_offset == 3 and img.pixels[2, 0] == 7
    ps = vm.project_all(vm.Volume(np.zeros((230, 512, 512), np.uint8)))        # :36-41
    assert (ps.diag.width, ps.diag.height) == (741, 512) and (ps.anti.width, ps.anti.height) == (741, 512)


def test_mixed_formula_regression_on_device_images(cuda):
    """test_moments3d.py:116-147 restated: the +-45 degree recombination pinned
    on the device images (oracle 2D moments as the checker)."""
    for seed in range(5):
        v = vm.random((9, 7, 5), 8, seed)
        truth = oracle.naive(v.voxels, 4)
        ps = vm.project_all(v)
        dm = oracle.moments2d(ps.diag.pixels, 4)
        am = oracle.moments2d(ps.anti.pixels, 4, ai=-ps.anti.origin_offset)
        assert dm[(3, 1)] - am[(3, 1)] - 2 * truth[(0, 1, 3)] == 6 * truth[(2, 1, 1)]
        assert dm[(3, 1)] + am[(3, 1)] - 2 * truth[(3, 1, 0)] == 6 * truth[(1, 1, 2)]


def test_engine_equivalence_and_invariants(cuda):
    for seed in range(3):                                     # test_moments3d.py:54-72
        v = vm.random((12, 9, 15), 16, seed)
        assert vm.dpm_moments(v, 4).values == oracle.naive(v.voxels, 4)
    a, b = vm.random((5, 6, 7), 8, 1), vm.random((5, 6, 7), 8, 2)            # linearity :96-102
    s = vm.Volume((a.voxels.astype(np.uint16) + b.voxels).astype(np.uint16))
    ta, tb, ts = (vm.dpm_moments(x, 6) for x in (a, b, s))
    assert all(ts[k] == ta[k] + tb[k] for k in ts.values)
    v = vm.random((6, 5, 4), 8, seed=3)                       # relabel :88-93
    vp = vm.Volume(np.ascontiguousarray(v.voxels.transpose(2, 0, 1)))
    t, tp = vm.dpm_moments(v, 6), vm.dpm_moments(vp, 6)
    assert all(val == t[(r, p, q)] for (p, q, r), val in tp.items())


def test_overflow_envelope_and_order_errors(cuda):
    v = vm.random((3, 200, 200), 16, seed=0)                  # :234-237 tall-thin 16-bit
    assert vm.dpm_moments(v, 4).values == oracle.naive(v.voxels, 4)
    with pytest.raises(ValueError, match="order"):
        vm.dpm_moments(vm.uniform((2, 2, 2), 1), 7)


def test_inconsistency_detected_on_corrupted_image(cuda):
    """test_moments3d.py:168-184 restated on the device pipeline: a projection
    route that disagrees must raise InconsistencyError naming the disagreement."""
    v = torch.from_numpy(vm.random((8, 8, 8), 8, seed=1).voxels.copy()).cuda()
    imgs = engine.project(v, 5)
    imgs[0][0, 0, 0] += 1
    acc = engine.moments2d_images(v, imgs, 4)
    res = engine.derive(acc, 4, kind="images")
    torch.cuda.synchronize()
    from paper_2012_08099_b200.moments3d import raise_status
    with pytest.raises(InconsistencyError, match="disagree"):
        raise_status(int(res.status[0]))


def test_batch_and_streaming_match_resident(cuda):
    rng = np.random.default_rng(7)
    batch = rng.integers(0, 256, size=(5, 24, 16, 64), dtype=np.uint8)
    got = vm.dpm_moments_batch(batch, 6)
    for b in range(5):
        assert got[b].values == oracle.naive(batch[b], 6)
    from paper_2012_08099_b200.streaming import HostStreamer
    vol = torch.from_numpy(rng.integers(0, 65536, size=(100, 40, 72), dtype=np.uint16)).pin_memory()
    hs = HostStreamer(tuple(vol.shape), vol.dtype, 6, chunk_planes=16)
    res = hs.moments(vol)
    torch.cuda.synchronize()
    assert dict(zip(vm.moment_indices(6), _ints(res))) == oracle.naive(vol.numpy(), 6)


def test_zslab_composition_on_device(cuda):
    vol = engine.synth_noise(512, 96, 0, 200, 3)
    whole = _ints(engine.moments(vol, 6))
    for splits in ((0, 200), (0, 64, 200), (0, 7, 100, 129, 200)):
        acc = None
        for z0, z1 in zip(splits, splits[1:]):
            part = engine.moments2d_partial(vol[z0:z1], 6, z0=z0)
            if acc is None:
                acc = part
            else:
                engine.acc_add(acc, part)
        assert _ints(engine.derive(acc, 6, kind=engine.acc_kind(vol, 6))) == whole, splits


def test_cfg5_full_volume_exact(cuda):
    """The headline config at full size: 2048^3 uint16, order 6, against the
    oracle on the same bytes, plus image-mass consistency."""
    vol = engine.synth_noise(2048, 2048, 0, 2048, 5)
    res = engine.moments(vol, 6)
    torch.cuda.synchronize()
    assert int(res.status[0]) == 0
    host = vol.cpu().numpy()
    oracle.set_threads(oracle.max_threads())
    want = oracle.dpm(host, 6)
    assert dict(zip(vm.moment_indices(6), _ints(res))) == want
    assert want[(0, 0, 0)] == int(host.sum(dtype=np.uint64))


def test_cfg5_full_size_projection_rows_bit_exact(cuda):
    """Projection verify mode at full size: the headline pass's
    images of the 2048^3 volume -- the layout-T image set the moments pipeline
    builds (engine.project_profile) -- compared bit for bit with the oracle's
    projection of the x/z-exchanged volume, on image rows y in 0-7, 1024-1031
    and 2040-2047 (every image except the y-summed profile is per row y; YZ is
    stored [x][y], so those rows are its columns)."""
    vol = engine.synth_noise(2048, 2048, 0, 2048, 5)
    assert engine.acc_kind(vol, 6) == "profile_t"
    imgs, _ = engine.project_profile(vol, 6)
    torch.cuda.synchronize()
    ys = np.r_[0:8, 1024:1032, 2040:2048]
    sub = np.concatenate([vol[:, a:a + 8, :].cpu().numpy() for a in (0, 1024, 2040)], axis=1)   # (z, y, x) rows ys
    transposed = np.ascontiguousarray(sub.transpose(2, 1, 0))           # V'(x', y, z') = V(z', y, x')
    oracle.set_threads(oracle.max_threads())
    want = oracle.project(transposed, 7)
    for k in (0, 3, 4, 5, 6):                                           # [y][...] images
        got = imgs[k][0][torch.from_numpy(ys).cuda()].cpu().numpy().view(np.uint32).astype(np.int64)
        assert np.array_equal(got, want[k]), k
    got_yz = imgs[1][0][:, torch.from_numpy(ys).cuda()].cpu().numpy().view(np.uint32).astype(np.int64)
    assert np.array_equal(got_yz, want[1])


@pytest.mark.parametrize("order", [3, 4, 5, 6])
def test_derive_exactness_and_nonexact_flag(cuda, order):
    """Epilogue alone: exact results from a volume's limb accumulator (two
    volumes per call, one warp each); a +1 on one oblique 2D moment breaks
    an exact division and must raise DPM_ST_NONEXACT, never a wrong value."""
    rng = np.random.default_rng(order)
    vols = rng.integers(0, 65535, size=(2, 13, 11, 17)).astype(np.uint16)
    acc = engine.moments2d_partial(torch.from_numpy(vols).cuda(), order)
    assert engine.acc_kind(torch.from_numpy(vols), order) == "profile"   # classic layout: slot tags below
    res = engine.derive(acc, order)
    got = res.i128.cpu().numpy()
    idx = vm.moment_indices(order)
    for b in range(2):
        want = oracle.naive(vols[b], order)
        assert engine.i128_to_ints(got[b]) == [want[k] for k in idx]
    assert res.status.cpu().tolist() == [0, 0]
    # perturb DIAG (p=2, q=1) of volume 1: M_{1,1,1} = f/2 becomes non-integral
    K = order
    i21 = 2 * (K + 1) - 1 + 1
    bad = acc.clone()
    bad[1, 3, i21, 0] += 1
    st = engine.derive(bad, order).status.cpu().tolist()
    assert st[0] == 0 and st[1] & 2, st
    if order >= 5:
        # perturb X2P (p=4, q=1): the 3-unknown solve's division by 6 fails
        i41 = 4 * (K + 1) - 4 * 3 // 2 + 1
        bad = acc.clone()
        bad[0, 5, i41, 0] += 1
        st = engine.derive(bad, order).status.cpu().tolist()
        assert st[0] & 2 and st[1] == 0, st


@pytest.mark.parametrize("order", [0, 2, 3, 4, 6])
def test_image_moments_2d(cuda, order):
    """Device 2D moments of stand-alone images == the direct definition
    (stored coordinates, origin carried) and, after shift_origin, the moments
    about the logical origin (ANTI's N-1)."""
    rng = np.random.default_rng(40 + order)
    px = rng.integers(0, 2**32, size=(7, 13), dtype=np.uint64)
    got = vm.image_moments(px, order)
    want = {(p, q): sum(int(px[j, i]) * i ** p * j ** q for j in range(7) for i in range(13))
            for p in range(order + 1) for q in range(order + 1 - p)}
    assert got.values == want and got.order == order
    v = vm.random((6, 5, 4), 16, seed=order)
    anti = vm.project(v, vm.Orientation.ANTI)
    m = vm.shift_origin(vm.brute_force_2d(anti, max(order, 1)), anti.origin_offset)
    n = v.dims[2]
    logical = {}
    vox = v.voxels.astype(object)
    for p in range(max(order, 1) + 1):
        for q in range(max(order, 1) + 1 - p):
            logical[(p, q)] = sum(vox[z, y, x] * (x - z) ** p * y ** q for z in range(n) for y in range(5) for x in range(6))
    assert m.values == logical


def test_image_moments_2d_errors(cuda):
    with pytest.raises(ValueError):
        vm.image_moments(np.zeros((3, 3, 3)), 3)
    with pytest.raises(ValueError):
        vm.image_moments(np.full((3, 3), -1), 3)
    with pytest.raises(ValueError):
        vm.image_moments(np.ones((3, 3)), 7)
    with pytest.raises(OverflowError):
        vm.image_moments(np.full((4000, 4000), 2**32 - 1, dtype=np.uint64), 6)


@pytest.mark.parametrize("order", [3, 4, 5, 6])
@pytest.mark.parametrize("shape,dt", [((9, 7, 5), np.uint8), ((13, 11, 203), np.uint16), ((5, 300, 4), np.uint16),
                                      ((20, 16, 264), np.int16)])
def test_direct_engines_naive_and_factored(cuda, order, shape, dt):
    """The reference's direct engines on the device (csrc/direct3d.cu): exact
    like the oracle's direct sum, for every dtype and shape, batch included."""
    rng = np.random.default_rng(order + sum(shape))
    if dt == np.int16:
        vol = rng.integers(-1024, 3072, size=shape).astype(np.int16)
        want = oracle.naive((vol.astype(np.int32) + 1024).astype(np.uint16), order)
        for method in (0, 1):
            import ctypes
            v = torch.from_numpy(vol).cuda()
            d = engine.make_desc(v, 1024)
            wsb = int(nat.lib().dpm_direct_workspace_bytes(ctypes.byref(d), order))
            ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
            out = torch.empty((1, len(want), 2), dtype=torch.int64, device="cuda")
            assert nat.lib().dpm_direct_moments(ctypes.byref(d), v.data_ptr(), order, method, ws.data_ptr(), wsb,
                                                out.data_ptr(), None, None) == 0
            torch.cuda.synchronize()
            assert engine.i128_to_ints(out[0].cpu().numpy()) == [want[k] for k in vm.moment_indices(order)]
        return
    vol = rng.integers(0, np.iinfo(dt).max + 1, size=shape).astype(dt)
    v = vm.Volume(vol)
    want = oracle.naive(vol, order)
    assert vm.naive_moments(v, order).values == want
    assert vm.factored_moments(v, order).values == want
    assert vm.dpm_moments(v, order).values == want


def test_direct_engines_full_width_exact(cuda):
    """2048-wide 16-bit volumes at order 4, where the reference's naive and
    factored engines raise OverflowError (moments3d.py:121-127, 158-161): exact
    here, equal to the projection engine."""
    vol = engine.synth_noise(2048, 64, 0, 8, 5).cpu().numpy()
    v = vm.Volume(vol)
    d = vm.dpm_moments(v, 4).values
    assert vm.naive_moments(v, 4).values == d and vm.factored_moments(v, 4).values == d
