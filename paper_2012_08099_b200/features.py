"""Derived features of exact 3D moments.

Host post-pass on a ``MomentTensor3`` -- O(#moments) work, nothing to put on
the device.  Same names, fields, arguments and errors as the reference
(features.py:19-146, harness.feature_report :22-59), one difference in how
the central moments are evaluated:

* ``central_moments`` -- the reference expands
  mu_pqr = sum C(p,a)C(q,b)C(r,c) (-cx)^(p-a)(-cy)^(q-b)(-cz)^(r-c) M_abc in
  float64 and documents ~1e-9 relative cancellation error.  Here the same
  expansion is evaluated EXACTLY: with S = M000 and the integer first moments
  Mx, My, Mz, S^(p+q+r) mu_pqr is an integer,
      sum C(p,a)C(q,b)C(r,c) (-Mx)^(p-a) (-My)^(q-b) (-Mz)^(r-c) S^(a+b+c) M_abc,
  so mu_pqr is that integer over S^(p+q+r), rounded once to float64.  The
  values agree with the reference within its stated tolerance and are the
  correctly rounded central moments.
* ``centroid``, ``normalize_scale``, ``apply_spacing``, ``shape_features``
  follow the reference formulas (float64; deterministic eigen-axis signs).
"""
from __future__ import annotations

from dataclasses import dataclass
from fractions import Fraction
from math import comb, sqrt

import numpy as np

from .errors import InconsistencyError
from .moments3d import ENGINES, MomentTensor3, moment_indices


@dataclass(frozen=True)
class CentralMoments3:
    """Central moments mu[p][q][r] about the centroid, order <= K."""

    order: int
    mu: dict[tuple[int, int, int], float]
    centroid: tuple[float, float, float]

    def __getitem__(self, pqr: tuple[int, int, int]) -> float:
        return self.mu[pqr]


@dataclass(frozen=True)
class ShapeFeatures:
    """Second-order shape summary: covariance (mass-normalised second central
    moments), eigenvalues (descending), axes (rows, unit, sign-fixed),
    elongation (l1/l2, l2/l3) and radius of gyration sqrt(trace)."""

    covariance: np.ndarray
    eigenvalues: tuple[float, float, float]
    axes: np.ndarray
    elongation: tuple[float, float]
    radius_of_gyration: float


def _mass(m: MomentTensor3) -> int:
    s = m[(0, 0, 0)]
    if s <= 0:
        raise ValueError("centroid undefined for zero total mass")
    return s


def centroid(m: MomentTensor3) -> tuple[float, float, float]:
    """(M100, M010, M001) / M000 (exact integer ratios, correctly rounded)."""
    s = _mass(m)
    return (m[(1, 0, 0)] / s, m[(0, 1, 0)] / s, m[(0, 0, 1)] / s)


def central_moments(m: MomentTensor3) -> CentralMoments3:
    """Central moments from raw moments, evaluated exactly (see module doc)."""
    s = _mass(m)
    mx, my, mz = m[(1, 0, 0)], m[(0, 1, 0)], m[(0, 0, 1)]
    k = m.order
    # per-axis binomial factors C(n, a) (-M1)^(n-a) S^a, reused across indices
    def axis_terms(m1):
        return [[comb(n, a) * (-m1) ** (n - a) * s ** a for a in range(n + 1)] for n in range(k + 1)]
    tx, ty, tz = axis_terms(mx), axis_terms(my), axis_terms(mz)
    mu = {}
    for (p, q, r) in moment_indices(k):
        num = 0
        for a in range(p + 1):
            for b in range(q + 1):
                fab = tx[p][a] * ty[q][b]
                for c in range(r + 1):
                    num += fab * tz[r][c] * m[(a, b, c)]
        mu[(p, q, r)] = float(Fraction(num, s ** (p + q + r)))
    return CentralMoments3(k, mu, centroid(m))


def normalize_scale(cm: CentralMoments3) -> dict[tuple[int, int, int], float]:
    """Scale invariants eta_pqr = mu_pqr / mu_000^((p+q+r)/3 + 1)."""
    mu0 = cm.mu[(0, 0, 0)]
    if mu0 <= 0:
        raise ValueError("scale normalization undefined for zero total mass")
    return {key: cm.mu[key] / mu0 ** (sum(key) / 3.0 + 1.0) for key in moment_indices(cm.order)}


def apply_spacing(cm: CentralMoments3, sx: float, sy: float, sz: float) -> CentralMoments3:
    """Voxel -> physical coordinates: mu'_pqr = sx^(1+p) sy^(1+q) sz^(1+r) mu_pqr."""
    if sx <= 0 or sy <= 0 or sz <= 0:
        raise ValueError(f"spacing components must be > 0, got {(sx, sy, sz)}")
    mu = {(p, q, r): sx ** (1 + p) * sy ** (1 + q) * sz ** (1 + r) * v for (p, q, r), v in cm.mu.items()}
    cx, cy, cz = cm.centroid
    return CentralMoments3(cm.order, mu, (cx * sx, cy * sy, cz * sz))


def shape_features(cm: CentralMoments3) -> ShapeFeatures:
    """Principal axes, elongation and radius of gyration from second-order mu."""
    mu0 = cm.mu[(0, 0, 0)]
    if mu0 <= 0:
        raise ValueError("shape features undefined for zero total mass")
    idx = [(2, 0, 0), (1, 1, 0), (1, 0, 1), (0, 2, 0), (0, 1, 1), (0, 0, 2)]
    c200, c110, c101, c020, c011, c002 = (cm[k] for k in idx)
    cov = np.array([[c200, c110, c101], [c110, c020, c011], [c101, c011, c002]]) / mu0
    w, v = np.linalg.eigh(cov)
    if w[0] < -1e-9 * max(w[-1], 1.0):
        raise InconsistencyError(f"covariance is not positive semi-definite: {w}")
    desc = np.argsort(w)[::-1]
    lam = w[desc]
    axes = np.ascontiguousarray(v[:, desc].T)
    for row in axes:                         # sign rule: largest-magnitude component positive
        if row[int(np.argmax(np.abs(row)))] < 0:
            row *= -1.0
    l1, l2, l3 = (float(x) for x in lam)
    elong = (l1 / l2 if l2 > 0 else float("inf"), l2 / l3 if l3 > 0 else float("inf"))
    return ShapeFeatures(covariance=cov, eigenvalues=(l1, l2, l3), axes=axes, elongation=elong,
                         radius_of_gyration=sqrt(max(l1 + l2 + l3, 0.0)))


def _key(pqr) -> str:
    return "".join(str(i) for i in pqr)


def feature_report(volume, order: int, engine: str = "dpm", spacing=None) -> dict:
    """Moments and derived features as a deterministic JSON-ready dict with
    the reference's keys (harness.feature_report, harness.py:22-59)."""
    return report_from_tensor(volume, ENGINES[engine](volume, order), order, engine, spacing)


def report_from_tensor(volume, tensor: MomentTensor3, order: int, engine: str, spacing=None) -> dict:
    """``feature_report`` of already computed moments (e.g. a streamed file)."""
    cm = central_moments(tensor)
    eta = normalize_scale(cm)
    idx = moment_indices(order)
    use = tuple(spacing if spacing is not None else volume.spacing)
    report = {
        "input": {"dims": list(volume.dims), "bit_depth": volume.bit_depth, "spacing": list(use)},
        "engine": engine,
        "order": order,
        "raw_moments": {_key(k): val for k, val in tensor.items()},
        "centroid": list(cm.centroid),
        "central_moments": {_key(k): cm.mu[k] for k in idx},
        "normalized_moments": {_key(k): eta[k] for k in idx},
    }
    if use != (1.0, 1.0, 1.0):
        phys = apply_spacing(cm, *use)
        report["physical_central_moments"] = {_key(k): phys.mu[k] for k in idx}
    sf = shape_features(cm)
    report["shape"] = {
        "covariance": [[float(x) for x in row] for row in sf.covariance],
        "eigenvalues": list(sf.eigenvalues),
        "principal_axes": [[float(x) for x in row] for row in sf.axes],
        "elongation": list(sf.elongation),
        "radius_of_gyration": sf.radius_of_gyration,
    }
    return report
