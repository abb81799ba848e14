"""Loaders for the committed golden fixtures (generated from the reference by
tests/golden/make_golden.py; the GPU box reads only these files)."""
from __future__ import annotations

import hashlib
import json
import os
from functools import lru_cache

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ORIENTATIONS = ("xy", "yz", "zx", "diag", "anti")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@lru_cache(maxsize=1)
def projections():
    z = np.load(os.path.join(GOLDEN, "projections.npz"))
    vols, imgs = {}, {}
    for key in z.files:
        parts = key.split("__")
        if parts[0] == "vol":
            vols[parts[1]] = z[key]
        else:
            imgs[(parts[1], parts[2])] = z[key]
    return vols, imgs


def parse_moments(d: dict) -> dict[tuple[int, int, int], int]:
    return {tuple(int(c) for c in k.split(",")): int(v) for k, v in d.items()}


@lru_cache(maxsize=1)
def moments():
    with open(os.path.join(GOLDEN, "moments.json")) as fh:
        return json.load(fh)["volumes"]


@lru_cache(maxsize=1)
def configs():
    with open(os.path.join(GOLDEN, "configs.json")) as fh:
        return json.load(fh)["configs"]


def extra_volume(name: str) -> np.ndarray:
    """Volumes recorded in moments.json without stored voxels (re-created from
    the reference's own generator stream, volume.py:220-227)."""
    if name == "random_64_seed1":
        v = np.random.default_rng(1).integers(0, 256, size=(64, 64, 64), dtype=np.uint8)
    elif name == "random16bit_3x200x200":
        v = np.random.default_rng(0).integers(0, 65536, size=(200, 200, 3), dtype=np.uint16)
    else:
        raise KeyError(name)
    assert sha(v) == moments()[name]["voxels_sha256"], name
    return v


def volume_for(name: str) -> np.ndarray:
    vols, _ = projections()
    return vols[name] if name in vols else extra_volume(name)
