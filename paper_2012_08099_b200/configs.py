"""Seeded synthetic stand-ins for the five BASELINE.json configs.

The paper's datasets (NPS NRRD volumes, the slicer MRI) are not available, so
every config is generated from a seed; the interpretations of BASELINE.json's
wording are pinned here.  Parity never depends on these choices: the GPU and
the oracle always consume the identical voxel bytes.

cfg1  64^3 uint8, i.i.d. uniform 0..255 == reference volume.random((64,)*3, 8, seed)
      (volume.py:220-227).
cfg2  256^3 uint16 MRI-like phantom: three nested ellipsoids painted largest
      first with intensities 200 / 800 / 1500.  Outer centre ~ U[0.4n, 0.6n]^3,
      outer semi-axes ~ U[0.2n, 0.3n]^3 (all inside the middle 60 % of the grid);
      each inner ellipsoid's centre is its parent's plus U[-0.03n, 0.03n]^3 and
      its semi-axes are the parent's times U[0.4, 0.7]^3.  Then Gaussian noise
      sigma = 30, rounded half-to-even, clipped to 0..4095.
cfg3  512^3 int16 CT-like: air -1024; a centred body ellipsoid (centre
      n/2 + U[-0.02n, 0.02n]^3, semi-axes ~ U[0.3n, 0.45n]^3) whose voxels are
      i.i.d. integers U{-100..100}; 20 spheres with radius U[5, 40] and centres
      uniform in the body's bounding box, each a constant integer U{300..3000}
      HU, painted in order; clipped to -1024..3071.  Moments are taken of
      value + 1024 (uint16 range 0..4095), offset applied on the device.
cfg4  B binary uint8 128^3 volumes; volume i uses seed (seed * 1_000_003 + i):
      rotation R uniform on SO(3) (QR of a Gaussian 3x3, sign-fixed, det +1),
      semi-axes a ~ U[10, 60]^3, centre 63.5 + U[-20, 20]^3; voxel p is 1 iff
      sum_k ((R^T (p - c))_k / a_k)^2 <= 1 (the volume.ellipsoid convention,
      volume.py:230-242, with a rotation).
cfg5  2048^3 uint16 smooth lattice value noise, generated on the device per
      global z plane (csrc/synth.cu); ``noise_slab_numpy`` reproduces it
      bit for bit on the host.
"""
from __future__ import annotations

import numpy as np

CFG_SHAPES = {1: (64, 64, 64), 2: (256, 256, 256), 3: (512, 512, 512), 4: (128, 128, 128), 5: (2048, 2048, 2048)}
CFG_ORDER = {1: 3, 2: 3, 3: 4, 4: 3, 5: 6}
CFG_OFFSET = {3: 1024}


def cfg1(seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, 256, size=(64, 64, 64), dtype=np.uint8)


def _paint_ellipsoid(grid, center, axes, value, z_chunk=64, rot=None):
    n, m, l = grid.shape
    cx, cy, cz = center
    a, b, c = axes
    x = np.arange(l, dtype=np.float64) - cx
    y = np.arange(m, dtype=np.float64) - cy
    z0 = max(0, int(np.floor(cz - c)) - 1)
    z1 = min(n, int(np.ceil(cz + c)) + 2)
    for zs in range(z0, z1, z_chunk):
        ze = min(z1, zs + z_chunk)
        z = np.arange(zs, ze, dtype=np.float64) - cz
        q = (z[:, None, None] / c) ** 2 + (y[None, :, None] / b) ** 2 + (x[None, None, :] / a) ** 2
        grid[zs:ze][q <= 1.0] = value


def cfg2(seed: int = 0, n: int = 256) -> np.ndarray:
    rng = np.random.default_rng(seed)
    grid = np.zeros((n, n, n), dtype=np.float64)
    centre = rng.uniform(0.4 * n, 0.6 * n, size=3)
    axes = rng.uniform(0.2 * n, 0.3 * n, size=3)
    for value in (200.0, 800.0, 1500.0):
        _paint_ellipsoid(grid, centre, axes, value)
        centre = centre + rng.uniform(-0.03 * n, 0.03 * n, size=3)
        axes = axes * rng.uniform(0.4, 0.7, size=3)
    out = np.empty((n, n, n), dtype=np.uint16)
    for zs in range(0, n, 32):
        noisy = grid[zs:zs + 32] + rng.normal(0.0, 30.0, size=grid[zs:zs + 32].shape)
        out[zs:zs + 32] = np.clip(np.rint(noisy), 0, 4095).astype(np.uint16)
    return out


def cfg3(seed: int = 0, n: int = 512) -> np.ndarray:
    rng = np.random.default_rng(seed)
    grid = np.full((n, n, n), -1024, dtype=np.int16)
    centre = n / 2 + rng.uniform(-0.02 * n, 0.02 * n, size=3)
    axes = rng.uniform(0.3 * n, 0.45 * n, size=3)
    body = np.zeros((n, n, n), dtype=bool)
    cx, cy, cz = centre
    a, b, c = axes
    x = np.arange(n, dtype=np.float64) - cx
    y = np.arange(n, dtype=np.float64) - cy
    for zs in range(0, n, 32):
        z = np.arange(zs, zs + 32, dtype=np.float64) - cz
        q = (z[:, None, None] / c) ** 2 + (y[None, :, None] / b) ** 2 + (x[None, None, :] / a) ** 2
        body[zs:zs + 32] = q <= 1.0
    for zs in range(0, n, 32):
        sl = body[zs:zs + 32]
        tissue = rng.integers(-100, 101, size=sl.shape, dtype=np.int16)
        g = grid[zs:zs + 32]
        g[sl] = tissue[sl]
    lo = np.maximum(centre - axes, 0)
    hi = np.minimum(centre + axes, n - 1)
    for _ in range(20):
        r = rng.uniform(5, 40)
        sc = rng.uniform(lo, hi)
        hu = int(rng.integers(300, 3001))
        _paint_ellipsoid(grid, sc, (r, r, r), hu)
    np.clip(grid, -1024, 3071, out=grid)
    return grid


def cfg4_params(count: int = 1024, seed: int = 0) -> np.ndarray:
    """[count, 15] float64 rows: centre (3), semi-axes (3), rotation R row-major (9)."""
    out = np.empty((count, 15), dtype=np.float64)
    for i in range(count):
        rng = np.random.default_rng(seed * 1_000_003 + i)
        g = rng.normal(size=(3, 3))
        q, r = np.linalg.qr(g)
        q = q * np.sign(np.diag(r))[None, :]
        if np.linalg.det(q) < 0:
            q[:, 0] = -q[:, 0]
        axes = rng.uniform(10, 60, size=3)
        centre = 63.5 + rng.uniform(-20, 20, size=3)
        out[i, 0:3] = centre
        out[i, 3:6] = axes
        out[i, 6:15] = q.ravel()
    return out


def cfg4_volume_numpy(params_row: np.ndarray, n: int = 128) -> np.ndarray:
    """One config-4 volume on the host (the CPU-baseline leg and tests)."""
    c = params_row[0:3]
    a = params_row[3:6]
    R = params_row[6:15].reshape(3, 3)
    idx = np.arange(n, dtype=np.float64)
    z, y, x = np.meshgrid(idx, idx, idx, indexing="ij")
    d = np.stack([x - c[0], y - c[1], z - c[2]], axis=-1)
    u = d @ R  # (R^T d)_k = sum_i d_i R[i, k]
    q = ((u / a) ** 2).sum(axis=-1)
    return (q <= 1.0).astype(np.uint8)


def cfg4_device(params: np.ndarray, n: int = 128, device="cuda", chunk: int = 64):
    """The config-4 batch generated on the device with torch ([B, n, n, n] uint8).

    Same formula as cfg4_volume_numpy in float64; data generation only, not
    part of the timed path."""
    import torch

    B = params.shape[0]
    out = torch.empty((B, n, n, n), dtype=torch.uint8, device=device)
    idx = torch.arange(n, dtype=torch.float64, device=device)
    z, y, x = torch.meshgrid(idx, idx, idx, indexing="ij")
    pos = torch.stack([x, y, z], dim=-1)  # [n,n,n,3]
    P = torch.as_tensor(params, dtype=torch.float64, device=device)
    for s in range(0, B, chunk):
        p = P[s:s + chunk]
        c = p[:, 0:3]
        a = p[:, 3:6]
        R = p[:, 6:15].reshape(-1, 3, 3)
        for b in range(p.shape[0]):
            d = pos - c[b]
            u = d @ R[b]
            q = ((u / a[b]) ** 2).sum(dim=-1)
            out[s + b] = (q <= 1.0).to(torch.uint8)
    return out


# ---- config 5: integer value noise (bit-identical mirror of csrc/synth.cu) ----

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _mix64(z: np.ndarray) -> np.ndarray:
    z = z + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def _lattice(seed: int, o: int, cx, cy, cz) -> np.ndarray:
    with np.errstate(over="ignore"):
        h = np.uint64(seed) ^ (np.uint64(o) << np.uint64(56))
        h = _mix64(h ^ (cx.astype(np.uint64) * np.uint64(0x8CB92BA72F3D8DD7)))
        h = _mix64(h ^ (cy.astype(np.uint64) * np.uint64(0xA24BAED4963EE407)))
        h = _mix64(h ^ (cz.astype(np.uint64) * np.uint64(0x9FB21C651E98DF25)))
    return h >> np.uint64(48)


def _sweight(f: np.ndarray, S: int) -> np.ndarray:
    f = f.astype(np.int64)
    return ((f * f * (3 * S - 2 * f)) * 65536 // (S * S * S)).astype(np.uint64)


def noise_slab_numpy(L: int, M: int, z0: int, nz: int, seed: int) -> np.ndarray:
    """Host mirror of dpm_synth_noise_u16: [nz, M, L] uint16, planes z0..z0+nz-1.

    Separable evaluation of the same integer formula: the x-lerp is done once
    per lattice row, then rows are gathered per y (bit-identical to the
    per-voxel form ``noise_slab_numpy_direct``)."""
    out = np.empty((nz, M, L), dtype=np.uint16)
    one = np.uint64(65536)
    xs = np.arange(L, dtype=np.int64)
    ys = np.arange(M, dtype=np.int64)
    with np.errstate(over="ignore"):
        for zi in range(nz):
            z = z0 + zi
            total = np.zeros((M, L), dtype=np.uint64)
            for o in range(4):
                S = 128 >> o
                cx, cy, cz = xs // S, ys // S, z // S
                wx = _sweight(xs - cx * S, S)[None, :]
                wy = _sweight(ys - cy * S, S)[:, None]
                wz = _sweight(np.array([z - cz * S]), S)[0]
                ncy, ncx = int(cy.max()) + 2, int(cx.max()) + 2
                rows = np.arange(ncy, dtype=np.int64)[:, None]
                cols = np.arange(ncx, dtype=np.int64)[None, :]
                c = []
                for dz in (0, 1):
                    H = _lattice(seed, o, cols, rows, np.full((ncy, ncx), cz + dz, dtype=np.int64))  # [ncy, ncx]
                    B = H[:, cx] * (one - wx) + H[:, cx + 1] * wx       # [ncy, L], < 2^32
                    c.append(B[cy] * (one - wy) + B[cy + 1] * wy)      # [M, L],  < 2^48
                v = (c[0] * (one - wz) + c[1] * wz) >> np.uint64(48)
                total += v << np.uint64(3 - o)
            out[zi] = (total // np.uint64(15)).astype(np.uint16)
    return out


def noise_slab_numpy_direct(L: int, M: int, z0: int, nz: int, seed: int) -> np.ndarray:
    """Per-voxel form of the noise (slow; cross-checks the separable form)."""
    z, y, x = np.meshgrid(np.arange(z0, z0 + nz, dtype=np.int64), np.arange(M, dtype=np.int64),
                          np.arange(L, dtype=np.int64), indexing="ij")
    total = np.zeros(z.shape, dtype=np.uint64)
    one = np.uint64(65536)
    with np.errstate(over="ignore"):
        for o in range(4):
            S = 128 >> o
            cx, cy, cz = x // S, y // S, z // S
            wx, wy, wz = _sweight(x - cx * S, S), _sweight(y - cy * S, S), _sweight(z - cz * S, S)
            c = []
            for dz in (0, 1):
                b = []
                for dy in (0, 1):
                    h0 = _lattice(seed, o, cx, cy + dy, cz + dz)
                    h1 = _lattice(seed, o, cx + 1, cy + dy, cz + dz)
                    b.append(h0 * (one - wx) + h1 * wx)
                c.append(b[0] * (one - wy) + b[1] * wy)
            v = (c[0] * (one - wz) + c[1] * wz) >> np.uint64(48)
            total += v << np.uint64(3 - o)
    return (total // np.uint64(15)).astype(np.uint16)
