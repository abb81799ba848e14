"""Pure-Python loop oracles for tiny volumes -- restatements of the reference
test oracles (pkg/tests/conftest.py:11-65), extended to the two order-5/6
images.  Test infrastructure only."""
from __future__ import annotations

import numpy as np


def project(voxels: np.ndarray, name: str) -> np.ndarray:
    """conftest.oracle_project (conftest.py:11-37) + x2p/x2m."""
    n, m, l = voxels.shape
    shapes = {"xy": (m, l), "yz": (n, m), "zx": (l, n), "diag": (m, l + n - 1), "anti": (m, l + n - 1),
              "x2p": (m, l + 2 * n - 2), "x2m": (m, l + 2 * n - 2)}
    out = np.zeros(shapes[name], np.int64)
    for z in range(n):
        for y in range(m):
            for x in range(l):
                v = int(voxels[z, y, x])
                if name == "xy":
                    out[y, x] += v
                elif name == "yz":
                    out[z, y] += v
                elif name == "zx":
                    out[x, z] += v
                elif name == "diag":
                    out[y, x + z] += v
                elif name == "anti":
                    out[y, x - z + n - 1] += v
                elif name == "x2p":
                    out[y, x + 2 * z] += v
                else:
                    out[y, x - 2 * z + 2 * (n - 1)] += v
    return out


def moments_3d(voxels: np.ndarray, order: int, z0: int = 0) -> dict[tuple[int, int, int], int]:
    """conftest.oracle_moments_3d (conftest.py:40-54), any order, exact."""
    n, m, l = voxels.shape
    out = {}
    for p in range(order + 1):
        for q in range(order + 1 - p):
            for r in range(order + 1 - p - q):
                acc = 0
                for z in range(n):
                    for y in range(m):
                        for x in range(l):
                            acc += int(voxels[z, y, x]) * x ** p * y ** q * (z + z0) ** r
                out[(p, q, r)] = acc
    return out


def moments_2d(pixels: np.ndarray, order: int, ai: int = 0, aj: int = 0) -> dict[tuple[int, int], int]:
    """conftest.oracle_moments_2d (conftest.py:57-65) about a logical origin."""
    h, w = pixels.shape
    return {(p, q): sum(int(pixels[j, i]) * (i + ai) ** p * (j + aj) ** q for j in range(h) for i in range(w))
            for p in range(order + 1) for q in range(order + 1 - p)}
