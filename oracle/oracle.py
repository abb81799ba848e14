"""ctypes front end of the C oracle (oracle/dpm_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Returns reference-shaped Python objects: images as int64 ``pixels[j, i]``
(projection.py:48-75) and moments as exact Python ints keyed by (p, q, r) in
``moment_indices`` order (moments3d.py:46-54).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from functools import lru_cache

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libdpm_oracle.so")

#: image order shared with the CUDA path: the reference's five plus the two
#: order-5/6 images (x+2z, y) and (x-2z, y)
IMAGE_NAMES = ("xy", "yz", "zx", "diag", "anti", "x2p", "x2m")

_DTYPE_CODE = {np.dtype(np.uint8): 1, np.dtype(np.uint16): 2, np.dtype(np.int16): 3}


def build() -> str:
    """Compile the oracle with its committed Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


@lru_cache(maxsize=1)
def load() -> ctypes.CDLL:
    if not os.path.exists(_LIB_PATH):
        build()
    lib = ctypes.CDLL(_LIB_PATH)
    i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
    lib.vmo_num_images.argtypes = [ctypes.c_int]
    lib.vmo_layout.argtypes = [i64, i64, i64, i64, ctypes.c_int] + [ctypes.POINTER(i64)] * 4
    lib.vmo_project.argtypes = [vp, ctypes.c_int, i32, i64, i64, i64, ctypes.c_int,
                                ctypes.POINTER(vp)]
    lib.vmo_moments2d.argtypes = [vp, i64, i64, i64, i64, ctypes.c_int, vp]
    lib.vmo_derive3d.argtypes = [vp, ctypes.c_int, vp]
    lib.vmo_derive3d.restype = ctypes.c_int
    lib.vmo_dpm.argtypes = [vp, ctypes.c_int, i32, i64, i64, i64, i64, ctypes.c_int, vp]
    lib.vmo_dpm.restype = ctypes.c_int
    lib.vmo_naive.argtypes = [vp, ctypes.c_int, i32, i64, i64, i64, i64, ctypes.c_int, vp]
    lib.vmo_naive_direct.argtypes = [vp, ctypes.c_int, i32, i64, i64, i64, i64, ctypes.c_int, vp]
    lib.vmo_set_threads.argtypes = [ctypes.c_int]
    lib.vmo_synth_noise_u16.argtypes = [vp, i64, i64, i64, i64, ctypes.c_uint64]
    return lib


def set_threads(n: int) -> None:
    load().vmo_set_threads(int(n))


def max_threads() -> int:
    return int(load().vmo_max_threads())


@lru_cache(maxsize=16)
def moment_indices(order: int) -> tuple[tuple[int, int, int], ...]:
    return tuple((p, q, r) for p in range(order + 1) for q in range(order + 1 - p)
                 for r in range(order + 1 - p - q))


def _idx2(order: int) -> list[tuple[int, int]]:
    return [(p, q) for p in range(order + 1) for q in range(order + 1 - p)]


def num_images(order: int) -> int:
    return int(load().vmo_num_images(order))


def layout(dims, img: int, z0: int = 0):
    """(W, H, ai, aj) of image ``img`` for a volume/slab of dims (L, M, N)."""
    L, M, N = dims
    out = [ctypes.c_int64() for _ in range(4)]
    load().vmo_layout(L, M, N, z0, img, *[ctypes.byref(o) for o in out])
    return tuple(int(o.value) for o in out)


def _vol(voxels: np.ndarray):
    v = np.ascontiguousarray(voxels)
    if v.ndim != 3 or v.dtype not in _DTYPE_CODE:
        raise ValueError(f"oracle takes a 3D uint8/uint16/int16 array, got {v.dtype} {v.shape}")
    n, m, l = v.shape
    return v, _DTYPE_CODE[v.dtype], (l, m, n)


def _from_i128(buf: np.ndarray) -> list[int]:
    lo = buf[:, 0].astype(np.uint64)
    hi = buf[:, 1]
    return [int(h) * (1 << 64) + int(l) for l, h in zip(lo.tolist(), hi.tolist())]


def _to_i128(values) -> np.ndarray:
    out = np.zeros((len(values), 2), dtype=np.int64)
    for k, v in enumerate(values):
        v = int(v) % (1 << 128)
        out[k, 0] = np.uint64(v & ((1 << 64) - 1)).view(np.int64)
        hi = v >> 64
        out[k, 1] = hi - (1 << 64) if hi >= (1 << 63) else hi
    return out


def project(voxels: np.ndarray, n_img: int = 5, offset: int = 0) -> list[np.ndarray]:
    """All ``n_img`` projection images, int64 ``pixels[j, i]`` (stored indices)."""
    v, code, dims = _vol(voxels)
    imgs = []
    for k in range(n_img):
        W, H, _, _ = layout(dims, k)
        imgs.append(np.zeros((H, W), dtype=np.int64))
    ptrs = (ctypes.c_void_p * n_img)(*[a.ctypes.data for a in imgs])
    load().vmo_project(v.ctypes.data, code, offset, *dims, n_img, ptrs)
    return imgs


def moments2d(pixels: np.ndarray, order: int, ai: int = 0, aj: int = 0) -> dict[tuple[int, int], int]:
    """Exact raw moments of one image about logical origin (stored i + ai, j + aj)."""
    px = np.ascontiguousarray(pixels, dtype=np.int64)
    h, w = px.shape
    buf = np.zeros((len(_idx2(order)), 2), dtype=np.int64)
    load().vmo_moments2d(px.ctypes.data, w, h, ai, aj, order, buf.ctypes.data)
    return dict(zip(_idx2(order), _from_i128(buf)))


def derive3d(m2d: list[dict], order: int):
    """Placement + cross-axis solve; returns (values dict, status)."""
    flat = []
    for block in m2d:
        flat.extend(block[pq] for pq in _idx2(order))
    buf = _to_i128(flat)
    out = np.zeros((len(moment_indices(order)), 2), dtype=np.int64)
    st = load().vmo_derive3d(buf.ctypes.data, order, out.ctypes.data)
    return dict(zip(moment_indices(order), _from_i128(out))), int(st)


def dpm(voxels: np.ndarray, order: int, z0: int = 0, offset: int = 0) -> dict[tuple[int, int, int], int]:
    """Whole DPM pipeline (project -> 2D moments -> derive), exact ints."""
    v, code, dims = _vol(voxels)
    out = np.zeros((len(moment_indices(order)), 2), dtype=np.int64)
    st = load().vmo_dpm(v.ctypes.data, code, offset, *dims, z0, order, out.ctypes.data)
    if st:
        raise RuntimeError(f"oracle derive3d status {st}")
    return dict(zip(moment_indices(order), _from_i128(out)))


def naive(voxels: np.ndarray, order: int, z0: int = 0, offset: int = 0) -> dict[tuple[int, int, int], int]:
    """Direct Eq. 2 sum, exact ints, factored row -> plane -> volume (the
    checker; factored_moments' evaluation order, moments3d.py:142-198)."""
    v, code, dims = _vol(voxels)
    out = np.zeros((len(moment_indices(order)), 2), dtype=np.int64)
    load().vmo_naive(v.ctypes.data, code, offset, *dims, z0, order, out.ctypes.data)
    return dict(zip(moment_indices(order), _from_i128(out)))


def naive_direct(voxels: np.ndarray, order: int, z0: int = 0, offset: int = 0) -> dict[tuple[int, int, int], int]:
    """Eq. 2 term by term -- every voxel times every moment's monomial, the
    naive O(n^3)-multiply direct sum (moments3d.py:78-139) -- exact ints.
    A CPU BASELINE for bench.py; tests pin it to ``naive``."""
    v, code, dims = _vol(voxels)
    out = np.zeros((len(moment_indices(order)), 2), dtype=np.int64)
    load().vmo_naive_direct(v.ctypes.data, code, offset, *dims, z0, order, out.ctypes.data)
    return dict(zip(moment_indices(order), _from_i128(out)))


def synth_noise(L: int, M: int, z0: int, nz: int, seed: int) -> np.ndarray:
    """[nz, M, L] uint16 slab of the config-5 noise volume (host copy of csrc/synth.cu)."""
    out = np.empty((nz, M, L), dtype=np.uint16)
    load().vmo_synth_noise_u16(out.ctypes.data, L, M, z0, nz, seed & ((1 << 64) - 1))
    return out
