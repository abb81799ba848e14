"""Generate the golden fixtures from the REFERENCE implementation.

Run here (the build container), where /root/reference exists:
    python tests/golden/make_golden.py
It imports the reference package read-only under the alias ``volmoments_ref``
(never copied) and records its outputs on seeded inputs:
  - projections.npz : reference project_all images (int64) of small volumes,
                      plus the volumes themselves
  - moments.json    : reference dpm_moments / naive_moments (exact ints as
                      strings) for K = 3, 4 on small and config-shaped volumes
  - configs.json    : reference dpm_moments of the config generators' outputs
                      (cfg1, cfg2, cfg3 after +1024, cfg4 volumes 0..3, a cfg5
                      slab), SHA-256 of their voxel bytes and of every
                      reference projection image
The GPU box has no /root/reference; tests read only these committed files.
"""
from __future__ import annotations

import hashlib
import importlib.util
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
REF_PKG = "/root/reference/pkg/src/volmoments"


def load_reference():
    spec = importlib.util.spec_from_file_location(
        "volmoments_ref", os.path.join(REF_PKG, "__init__.py"), submodule_search_locations=[REF_PKG])
    mod = importlib.util.module_from_spec(spec)
    sys.modules["volmoments_ref"] = mod
    spec.loader.exec_module(mod)
    return mod


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def small_volumes(ref):
    vols = {
        "uniform_2x2x2": ref.uniform((2, 2, 2), 1).voxels,
        "uniform_5x3x2": ref.uniform((5, 3, 2), 1).voxels,
        "delta_diag": ref.delta((4, 4, 4), (1, 0, 1), 7).voxels,
        "delta_anti": ref.delta((4, 4, 4), (0, 2, 3), 7).voxels,
        "delta_monomial": ref.delta((4, 5, 6), (1, 2, 3), 5).voxels,
        "random_16_seed7": ref.random((16, 16, 16), 8, seed=7).voxels,
        "random16bit_9x5x7": ref.random((9, 5, 7), 16, seed=3).voxels,
        "random_6x5x4_s11": ref.random((6, 5, 4), 8, seed=11).voxels,
        "random_6x5x4_s13": ref.random((6, 5, 4), 8, seed=13).voxels,
        "random_9x7x5_s0": ref.random((9, 7, 5), 8, seed=0).voxels,
        "random_5x5x5_s0": ref.random((5, 5, 5), 8, seed=0).voxels,
    }
    g = np.zeros((4, 4, 4), np.uint8)
    g[0, 0, 0] = 1
    g[3, 2, 1] = 2
    vols["two_voxel"] = g
    rng = np.random.default_rng(2012_08099)
    for k in range(16):
        dims = tuple(int(d) for d in rng.integers(1, 9, size=3))
        vols[f"hyp_{k}_{dims[0]}x{dims[1]}x{dims[2]}"] = ref.random(dims, 8, seed=k).voxels
    for s in range(3):
        vols[f"random16bit_12x9x15_s{s}"] = ref.random((12, 9, 15), 16, s).voxels
    return {k: np.ascontiguousarray(v) for k, v in vols.items()}


def moments_dict(t) -> dict:
    return {f"{p},{q},{r}": str(v) for (p, q, r), v in t.items()}


def main():
    ref = load_reference()
    from paper_2012_08099_b200 import configs as synth

    # 1. projections of small volumes
    vols = small_volumes(ref)
    arrays = {}
    for name, v in vols.items():
        ps = ref.project_all(ref.Volume(v.copy()))
        arrays[f"vol__{name}"] = v
        for o in ref.Orientation:
            arrays[f"img__{name}__{o.value}"] = ps[o].pixels
    np.savez_compressed(os.path.join(HERE, "projections.npz"), **arrays)

    # 2. moments (reference dpm + naive) of small / medium volumes
    mom = {}
    extra = {
        "random_64_seed1": ref.random((64, 64, 64), 8, seed=1).voxels,
        "random16bit_3x200x200": ref.random((3, 200, 200), 16, seed=0).voxels,
    }
    for name, v in list(vols.items()) + list(extra.items()):
        vol = ref.Volume(np.ascontiguousarray(v).copy())
        entry = {"shape": list(v.shape), "dtype": str(v.dtype), "voxels_sha256": sha(v)}
        for K in (3, 4):
            entry[f"dpm{K}"] = moments_dict(ref.dpm_moments(vol, K))
            entry[f"naive{K}"] = moments_dict(ref.naive_moments(vol, K))
        mom[name] = entry
    with open(os.path.join(HERE, "moments.json"), "w") as fh:
        json.dump({"source": "reference volmoments (dpm_moments, naive_moments)", "volumes": mom}, fh)
    # extra volumes are not stored: they are volume.random((64,)*3, 8, 1) and
    # volume.random((200, 200, 3), 16, 0), re-created in the tests and checked by sha256

    # 3. config generators -> reference outputs
    cfgs = {}

    def record(name, voxels_u16_or_u8, K, raw_sha, params):
        vol = ref.Volume(np.ascontiguousarray(voxels_u16_or_u8).copy())
        ps = ref.project_all(vol)
        cfgs[name] = {
            "params": params, "order": K, "voxels_sha256": raw_sha,
            "dpm": moments_dict(ref.dpm_moments(vol, K)),
            "images_sha256": {o.value: sha(ps[o].pixels) for o in ref.Orientation},
            "images_mass": {o.value: str(ps[o].mass) for o in ref.Orientation},
        }
        print(name, "done", flush=True)

    v1 = synth.cfg1(0)
    assert np.array_equal(v1, ref.random((64, 64, 64), 8, seed=0).voxels)
    record("cfg1", v1, 3, sha(v1), {"seed": 0})
    cfgs["cfg1"]["naive"] = moments_dict(ref.naive_moments(ref.Volume(v1.copy()), 3))
    v2 = synth.cfg2(0)
    record("cfg2", v2, 3, sha(v2), {"seed": 0})
    v3 = synth.cfg3(0)
    record("cfg3", (v3.astype(np.int32) + 1024).astype(np.uint16), 4, sha(v3), {"seed": 0, "offset": 1024})
    params = synth.cfg4_params(4, seed=0)
    for i in range(4):
        v4 = synth.cfg4_volume_numpy(params[i])
        record(f"cfg4_{i}", v4, 3, sha(v4), {"seed": 0, "index": i})
    v5 = synth.noise_slab_numpy(2048, 2048, 1000, 4, 5)
    record("cfg5_slab", v5, 4, sha(v5), {"L": 2048, "M": 2048, "z0": 1000, "nz": 4, "seed": 5})
    cfgs["cfg5_slab"]["naive3"] = moments_dict(ref.naive_moments(ref.Volume(v5.copy()), 3))
    with open(os.path.join(HERE, "configs.json"), "w") as fh:
        json.dump({"source": "reference volmoments on paper_2012_08099_b200.configs generators",
                   "configs": cfgs}, fh, indent=0)


if __name__ == "__main__":
    main()
