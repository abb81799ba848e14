"""Host-side logic of the package (no GPU)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2012_08099_b200 as vm
from paper_2012_08099_b200 import configs as synth, engine
from paper_2012_08099_b200.errors import InconsistencyError
from paper_2012_08099_b200.moments3d import raise_status


def test_moment_indices_match_reference_order():
    for K in (3, 4, 5, 6):
        idx = vm.moment_indices(K)
        assert idx == oracle.moment_indices(K) and list(idx) == sorted(idx)
    assert len(vm.moment_indices(3)) == 20 and len(vm.moment_indices(6)) == 84


def test_i128_and_limb_roundtrip():
    vals = [0, 1, -1, 2 ** 64 + 7, -(2 ** 100) + 3, 2 ** 126 - 1, -(2 ** 126)]
    pairs = np.array([[(v % (1 << 128)) & ((1 << 64) - 1), (v % (1 << 128)) >> 64] for v in vals], dtype=object)
    lo = np.array([int(x) for x in pairs[:, 0]], dtype=np.uint64).view(np.int64)
    hi = np.array([int(x) - (1 << 64) if int(x) >= (1 << 63) else int(x) for x in pairs[:, 1]], dtype=np.int64)
    assert engine.i128_to_ints(np.stack([lo, hi], axis=1)) == vals
    limbs = engine.ints_to_limbs(vals)
    assert engine.acc_to_ints(limbs).tolist() == vals
    # limb encodings add like the device atomics do (mod 2^64 per limb)
    s = (limbs.view(np.uint64) + limbs.view(np.uint64)).view(np.int64)
    assert engine.acc_to_ints(s).tolist() == [2 * v for v in vals]


def test_order_validation():
    for bad in (2, 7, 0, "4"):
        with pytest.raises(ValueError, match="order"):
            engine.check_order(bad)
    for ok in (3, 4, 5, 6):
        engine.check_order(ok)


def test_status_mapping():
    raise_status(0)
    with pytest.raises(InconsistencyError, match="disagree"):
        raise_status(1)
    with pytest.raises(InconsistencyError, match="remainder"):
        raise_status(2)
    with pytest.raises(InconsistencyError, match="mass"):
        raise_status(4)


def test_make_desc_strides_and_dtypes():
    t = torch.zeros((5, 6, 16), dtype=torch.uint16)
    d = engine.make_desc(t, offset=0, z0=7)
    assert (d.L, d.M, d.N, d.B, d.stride_y, d.stride_z, d.z0) == (16, 6, 5, 1, 16, 96, 7)
    b = torch.zeros((3, 5, 6, 16), dtype=torch.int16)
    d = engine.make_desc(b, offset=1024)
    assert (d.B, d.stride_b, d.dtype, d.offset) == (3, 480, 3, 1024)
    with pytest.raises(ValueError):
        engine.make_desc(torch.zeros((4, 4, 4), dtype=torch.float32))
    with pytest.raises(ValueError):
        engine.make_desc(torch.zeros((4, 4, 4), dtype=torch.uint8)[:, :, ::2])


def test_volume_model_matches_reference_contract():
    v = vm.uniform((2, 3, 4), 1)
    assert v.dims == (2, 3, 4) and v.mass == 24 and v.bit_depth == 8
    with pytest.raises(ValueError):
        v.voxels[0, 0, 0] = 2
    with pytest.raises(ValueError):
        vm.Volume(np.zeros((2, 2, 2), np.int16))
    r = vm.random((64, 64, 64), 8, seed=0)
    assert np.array_equal(r.voxels, synth.cfg1(0))


def test_noise_generators_agree():
    a = synth.noise_slab_numpy(160, 40, 250, 2, 9)
    assert np.array_equal(a, synth.noise_slab_numpy_direct(160, 40, 250, 2, 9))
    assert np.array_equal(a, oracle.synth_noise(160, 40, 250, 2, 9))


def test_compute_calls_fail_loudly_without_cuda():
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(Exception):
        vm.dpm_moments(vm.uniform((2, 2, 2), 1), 3)


def _brute2d(px, order, x0=0):
    """Pure-Python 2D moments about first-axis origin x0 (test restatement of
    the reference's direct definition, drt2d.py:177-193)."""
    h, w = px.shape
    out = {}
    for p in range(order + 1):
        for q in range(order + 1 - p):
            out[(p, q)] = sum(int(px[j, i]) * (i - x0) ** p * j ** q for j in range(h) for i in range(w))
    return out


def test_shift_origin_matches_direct_definition():
    from paper_2012_08099_b200.drt2d import Moments2D, shift_origin
    rng = np.random.default_rng(4)
    px = rng.integers(0, 1000, size=(5, 9))
    for order, off in [(3, 2), (4, 8), (6, 3)]:
        m = Moments2D(order, _brute2d(px, order), origin_offset=off)
        sh = shift_origin(m, off)
        assert sh.origin_offset == 0 and sh.order == order
        assert sh.values == _brute2d(px, order, x0=off)
        assert shift_origin(m, 0).values == m.values


def test_moments2d_type_mirrors_reference():
    from paper_2012_08099_b200.drt2d import Moments2D
    m = Moments2D(3, {(0, 0): 7, (1, 0): 3}, 2)
    assert m[(1, 0)] == 3 and m.mass == 7 and m.origin_offset == 2


def test_int16_offset_range_is_validated():
    """int16 + offset must land in 0..65535 (exact uint32 ray sums): a negative
    voxel without an offset, or an offset pushing values past 65535, is
    refused before any device work; unsigned voxels take no offset."""
    ok = torch.tensor([[[-1024, 3071]]], dtype=torch.int16)
    engine.make_desc(ok, offset=1024)
    with pytest.raises(ValueError, match="outside 0..65535"):
        engine.make_desc(ok, offset=0)
    with pytest.raises(ValueError, match="outside 0..65535"):
        engine.make_desc(torch.tensor([[[30000]]], dtype=torch.int16), offset=40000)
    with pytest.raises(ValueError, match="int16 input only"):
        engine.make_desc(torch.zeros((2, 2, 2), dtype=torch.uint16), offset=5)
    with pytest.raises(ValueError):
        engine.make_desc(ok, offset=200000)


def test_volmoments_dropin_surface():
    """``import volmoments`` resolves to this package: the reference's module
    names alias the engine's modules, the public names exist, and the only
    reference exports missing are the documented integral-route internals."""
    import volmoments
    import volmoments.moments3d
    import volmoments.projection
    from oracle import reference
    assert volmoments.moments3d is vm.moments3d and volmoments.projection is vm.projection
    assert volmoments.dpm_moments is vm.dpm_moments
    assert set(volmoments.moments3d.ENGINES) == {"naive", "factored", "dpm", "dpm_generic"}
    ref = reference.load()
    if ref is not None:
        missing = set(ref.__all__) - set(dir(volmoments))
        assert missing <= {"IntegralSet", "integrals", "moments_1d", "assemble_2d"}, missing
