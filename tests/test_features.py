"""Feature epilogue (centroid, central / normalised moments, spacing, shape):
known answers on exact oracle moments (CPU), agreement with the reference's
own feature code when it is importable (CPU), and the reference's
feature tests through the device engine (GPU)."""
import json
import os
import sys

import numpy as np
import pytest

import oracle
import paper_2012_08099_b200 as vm
from paper_2012_08099_b200.moments3d import MomentTensor3


def tensor(v, order):
    """Exact MomentTensor3 of a Volume from the C oracle (no GPU)."""
    return MomentTensor3(order, oracle.naive(v.voxels, order))


def mu_direct(v, order):
    """Direct-definition central moments in exact rational arithmetic."""
    from fractions import Fraction
    vox = v.voxels.astype(object)
    n, m, l = vox.shape
    s = int(v.voxels.sum(dtype=np.int64))
    zz, yy, xx = np.meshgrid(range(n), range(m), range(l), indexing="ij")
    c = [Fraction(int((vox * a).sum()), s) for a in (xx, yy, zz)]
    out = {}
    for (p, q, r) in vm.moment_indices(order):
        tot = Fraction(0)
        for (z, y, x), val in np.ndenumerate(vox):
            if val:
                tot += val * (x - c[0]) ** p * (y - c[1]) ** q * (z - c[2]) ** r
        out[(p, q, r)] = float(tot)
    return out


def test_centroid_known_answers():
    assert vm.centroid(tensor(vm.delta((4, 4, 4), (1, 2, 3), 9), 4)) == (1, 2, 3)
    assert vm.centroid(tensor(vm.uniform((2, 2, 2), 1), 4)) == (0.5, 0.5, 0.5)
    with pytest.raises(ValueError, match="zero"):
        vm.centroid(tensor(vm.uniform((2, 2, 2), 0), 4))


@pytest.mark.parametrize("order", [3, 4, 6])
def test_central_moments_exact(order):
    v = vm.random((6, 5, 4), 16, seed=order)
    cm = vm.central_moments(tensor(v, order))
    want = mu_direct(v, order)
    assert cm.mu == want                     # correctly rounded exact values, bit for bit
    d = vm.central_moments(tensor(vm.delta((5, 5, 5), (2, 1, 3), 7), order))
    assert d.mu[(0, 0, 0)] == 7 and all(val == 0.0 for key, val in d.mu.items() if sum(key) >= 1)


def test_normalize_spacing_shape():
    v = vm.random((16, 16, 16), 8, seed=0)
    cm = vm.central_moments(tensor(v, 4))
    eta = vm.normalize_scale(cm)
    assert eta[(0, 0, 0)] == 1.0 and all(abs(eta[k]) < 1e-12 for k in [(1, 0, 0), (0, 1, 0), (0, 0, 1)])
    assert vm.apply_spacing(cm, 1.0, 1.0, 1.0).mu == cm.mu
    out = vm.apply_spacing(cm, 2.0, 3.0, 0.5)
    assert out.mu[(1, 1, 1)] == pytest.approx(2.0**2 * 3.0**2 * 0.5**2 * cm.mu[(1, 1, 1)])
    with pytest.raises(ValueError, match="spacing"):
        vm.apply_spacing(cm, 1.0, -1.0, 1.0)
    sf = vm.shape_features(cm)
    assert sum(sf.eigenvalues) == pytest.approx(float(np.trace(sf.covariance)), rel=1e-9)
    assert np.allclose(sf.axes @ sf.axes.T, np.eye(3), atol=1e-9)
    for axis in sf.axes:
        assert axis[int(np.argmax(np.abs(axis)))] > 0
    a, b, c = 24.0, 18.0, 12.0
    e = vm.ellipsoid((52, 40, 28), (25.5, 19.5, 13.5), (a, b, c), 1)
    lam = vm.shape_features(vm.central_moments(tensor(e, 3))).eigenvalues
    assert lam[0] / lam[1] == pytest.approx((a / b) ** 2, rel=0.02)
    assert lam[1] / lam[2] == pytest.approx((b / c) ** 2, rel=0.02)


def _reference():
    from oracle import reference
    ref = reference.load()      # read-only, under the alias volmoments_ref
    if ref is None:
        pytest.skip("reference package not present")
    return ref


@pytest.mark.parametrize("dims,bits,seed", [((24, 20, 16), 8, 5), ((12, 9, 15), 16, 1), ((32, 32, 32), 8, 4)])
def test_features_agree_with_reference(dims, bits, seed):
    ref = _reference()
    rv = ref.random(dims, bits, seed=seed)
    ours_t = MomentTensor3(4, oracle.naive(rv.voxels, 4))
    ref_t = ref.dpm_moments(rv, 4)
    assert dict(ref_t.items()) == dict(ours_t.items())
    rc, oc = ref.central_moments(ref_t), vm.central_moments(ours_t)
    mass, ext = float(ref_t.mass), max(dims) / 2.0
    for k, val in rc.mu.items():      # the reference's stated float64 tolerance
        assert abs(val - oc.mu[k]) <= 1e-9 * max(mass * ext ** sum(k), 1.0), k
    assert rc.centroid == oc.centroid
    rs, os_ = ref.shape_features(rc), vm.shape_features(oc)
    assert np.allclose(rs.eigenvalues, os_.eigenvalues, rtol=1e-9)
    assert np.allclose(rs.axes, os_.axes, atol=1e-7)


@pytest.mark.gpu
def test_feature_report_through_device_engine(cuda):
    v = vm.Volume(vm.random((20, 18, 16), 8, seed=2).voxels, spacing=(1.0, 1.0, 0.5))
    rep = vm.feature_report(v, 4)
    assert rep["engine"] == "dpm" and rep["order"] == 4 and "physical_central_moments" in rep
    exact = oracle.naive(v.voxels, 4)
    assert rep["raw_moments"] == {"".join(map(str, k)): val for k, val in sorted(exact.items())}
    assert rep["central_moments"] == {"".join(map(str, k)): val
                                      for k, val in vm.central_moments(MomentTensor3(4, exact)).mu.items()}
    json.dumps(rep)   # JSON-ready
