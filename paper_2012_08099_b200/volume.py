"""Volume data model (reference volume.py:20-53) and the reference's small
synthetic generators (volume.py:199-270), kept so callers of the reference API
find the same names.  File loaders (load_raw/load_nrrd) are out of scope for
this hot-path build.

A volume is a dense grid of unsigned 8/16-bit intensities laid out x-fastest:
voxel (x, y, z) lives at flat offset x + L*(y + M*z), i.e. ``voxels[z, y, x]``.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_DTYPES = {8: np.dtype("<u1"), 16: np.dtype("<u2")}


@dataclass(frozen=True, eq=False)
class Volume:
    """Immutable 3D voxel grid with physical spacing (reference volume.py:20-53).

    voxels  -- uint8 or uint16 array of shape (N, M, L), i.e. [z, y, x]
    spacing -- physical units per voxel along (x, y, z); all > 0
    """

    voxels: np.ndarray
    spacing: tuple[float, float, float] = (1.0, 1.0, 1.0)

    def __post_init__(self):
        if self.voxels.ndim != 3:
            raise ValueError(f"voxel grid must be 3D, got {self.voxels.ndim}D")
        if self.voxels.dtype not in (np.uint8, np.uint16):
            raise ValueError(f"unsupported voxel dtype {self.voxels.dtype}; use uint8 or uint16")
        if len(self.spacing) != 3 or any(s <= 0 for s in self.spacing):
            raise ValueError(f"spacing components must be > 0, got {self.spacing}")
        self.voxels.setflags(write=False)

    @property
    def dims(self) -> tuple[int, int, int]:
        """(L, M, N) voxel counts along x, y, z."""
        n, m, l = self.voxels.shape
        return (l, m, n)

    @property
    def bit_depth(self) -> int:
        return 8 if self.voxels.dtype == np.uint8 else 16

    @property
    def mass(self) -> int:
        """Total intensity, exact."""
        return int(self.voxels.sum(dtype=np.int64))


def uniform(dims: tuple[int, int, int], value: int = 1, *, spacing=(1.0, 1.0, 1.0),
            bit_depth: int = 8) -> Volume:
    l, m, n = dims
    dtype = _DTYPES[bit_depth]
    if not 0 <= value <= np.iinfo(dtype).max:
        raise ValueError(f"value {value} does not fit {bit_depth}-bit intensities")
    return Volume(np.full((n, m, l), value, dtype=dtype), spacing)


def delta(dims: tuple[int, int, int], position: tuple[int, int, int], value: int = 1, *,
          spacing=(1.0, 1.0, 1.0), bit_depth: int = 8) -> Volume:
    """Single voxel of ``value`` at (x0, y0, z0), zeros elsewhere."""
    l, m, n = dims
    x0, y0, z0 = position
    if not (0 <= x0 < l and 0 <= y0 < m and 0 <= z0 < n):
        raise ValueError(f"delta position {position} outside dims {dims}")
    grid = np.zeros((n, m, l), dtype=_DTYPES[bit_depth])
    grid[z0, y0, x0] = value
    return Volume(grid, spacing)


def random(dims: tuple[int, int, int], bit_depth: int = 8, seed: int = 0, *,
           spacing=(1.0, 1.0, 1.0)) -> Volume:
    """Seed-deterministic uniform random intensities over the full bit range
    (same stream as the reference's volume.random, volume.py:220-227)."""
    l, m, n = dims
    dtype = _DTYPES[bit_depth]
    rng = np.random.default_rng(seed)
    grid = rng.integers(0, np.iinfo(dtype).max + 1, size=(n, m, l), dtype=dtype)
    return Volume(grid, spacing)


def ellipsoid(dims: tuple[int, int, int], center: tuple[float, float, float],
              semi_axes: tuple[float, float, float], value: int = 1, *,
              spacing=(1.0, 1.0, 1.0), bit_depth: int = 8) -> Volume:
    """Solid ellipsoid: voxels whose centres satisfy the implicit inequality."""
    l, m, n = dims
    cx, cy, cz = center
    a, b, c = semi_axes
    x = (np.arange(l) - cx) / a
    y = (np.arange(m) - cy) / b
    z = (np.arange(n) - cz) / c
    inside = (z[:, None, None] ** 2 + y[None, :, None] ** 2 + x[None, None, :] ** 2) <= 1.0
    return Volume(np.where(inside, value, 0).astype(_DTYPES[bit_depth]), spacing)


def synth(kind: str, dims: tuple[int, int, int], seed: int = 0, *, spacing=(1.0, 1.0, 1.0)) -> Volume:
    """Synthetic volume from a descriptor (the reference CLI's ``--synth``,
    volume.py:245-270): ``uniform:V``, ``delta:X,Y,Z,V``, ``random:BITDEPTH``,
    ``ellipsoid:CX,CY,CZ,A,B,C[,V]``; ``seed`` only feeds ``random``."""
    name, _, arg = kind.partition(":")
    builders = {
        "uniform": lambda: uniform(dims, int(arg or 1), spacing=spacing),
        "delta": lambda: _delta_from(arg, dims, spacing),
        "random": lambda: random(dims, int(arg or 8), seed, spacing=spacing),
        "ellipsoid": lambda: _ellipsoid_from(arg, dims, spacing),
    }
    if name not in builders:
        raise ValueError(f"unknown synth kind {name!r}")
    try:
        return builders[name]()
    except ValueError as exc:
        msg = str(exc)
        if "outside dims" in msg or "does not fit" in msg:
            raise
        raise ValueError(f"malformed synth descriptor {kind!r}") from exc


def _delta_from(arg: str, dims, spacing) -> Volume:
    x0, y0, z0, v = (int(t) for t in arg.split(","))
    return delta(dims, (x0, y0, z0), v, spacing=spacing)


def _ellipsoid_from(arg: str, dims, spacing) -> Volume:
    vals = [float(t) for t in arg.split(",")]
    if len(vals) < 6:
        raise ValueError("ellipsoid needs CX,CY,CZ,A,B,C")
    value = int(vals[6]) if len(vals) > 6 else 1
    return ellipsoid(dims, tuple(vals[0:3]), tuple(vals[3:6]), value, spacing=spacing)
