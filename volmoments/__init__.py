"""``volmoments`` -- the reference package's import name, backed by the B200 engine.

A drop-in for code written against the reference (``import volmoments as vm``;
``/root/reference/pkg/src/volmoments/__init__.py:10-38``): the same module
names (``volmoments.moments3d``, ``.projection``, ``.drt2d``, ``.volume``,
``.errors``, ``.counters``, ``.features``, ``.harness``, ``.cli``) resolve to the
modules of :mod:`paper_2012_08099_b200`, whose hot path -- projection pass,
exact 2D moments, 3D epilogue -- runs in the sm_100a CUDA kernels behind the
C ABI (include/dpm_b200.h).  There is no CPU fallback: without the CUDA
library and a GPU, compute calls raise.

Documented deviations from the reference:

* orders 3..6 are accepted (the reference accepts 3-4, moments3d.py:57-59);
* ``ENGINES`` holds the reference's three engines, all on the device --
  ``naive``, ``factored`` (exact direct sums, csrc/direct3d.cu) and ``dpm`` --
  plus ``dpm_generic`` (a second projection route); they are exact at every
  size inside the envelope, so the reference's OverflowError for 2048-wide
  16-bit naive/factored sums does not occur;
* the 1D-integral internals (``integrals``, ``IntegralSet``, ``moments_1d``,
  ``assemble_2d``, ``volmoments.exact``) are not provided: the device
  power-table kernel replaces the integral route (any order up to 6);
  a reference installation keeps its own and can add the CUDA engine to its
  registry with :func:`register`;
* ``counters=`` tallies the device method: P additions per voxel and Theta(n^2)
  row-power multiplications (the reference's integral route has Theta(n));
* the Python seams the reference's monkeypatch tests corrupt
  (``moments3d._cross_axis_moments``, ``project_subset`` inside
  ``dpm_moments``) do not exist: the epilogue runs on the device.
"""
from __future__ import annotations

import sys as _sys

import paper_2012_08099_b200 as _impl
from paper_2012_08099_b200 import (cli, counters, drt2d, errors, features, harness, moments3d, projection,
                                   volio, volume)

# volmoments.<module> is the engine's module itself (monkeypatching one patches both)
for _name, _mod in (("cli", cli), ("counters", counters), ("drt2d", drt2d), ("errors", errors),
                    ("features", features), ("harness", harness), ("moments3d", moments3d),
                    ("projection", projection), ("volume", volume), ("volio", volio)):
    _sys.modules[f"{__name__}.{_name}"] = _mod

from paper_2012_08099_b200 import (ANGLES, BenchReport, CentralMoments3, ENGINES, FormatError,  # noqa: E402
                                   InconsistencyError, MomentTensor3, Moments2D, OpCounters, Orientation,
                                   ProjectionImage, ProjectionSet, ShapeFeatures, Volume, VolumeMeta,
                                   apply_spacing, brute_force_2d, central_moments, centroid, count_ops, delta,
                                   dpm_moments, dpm_moments_batch, dpm_moments_file, ellipsoid, factored_moments,
                                   feature_report, naive_moments,
                                   load_nrrd, load_raw, meta_from_header_file, moment_indices, normalize_scale,
                                   project, project_all, project_subset, random, run_bench, shape_features,
                                   shift_origin, synth, uniform, verify_engines, write_pgm, write_raw)

__version__ = _impl.__version__


def register(engines: dict, name: str = "dpm_cuda") -> None:
    """Add the CUDA engine to a reference ``ENGINES`` registry (the reference
    side of INTEGRATION.md §2, ``moments3d.py:267-271``): the reference's
    ``harness.verify_engines`` / ``run_bench`` / ``count_ops`` and the CLI's
    ``--engine`` then run it beside its own CPU engines.  The engine takes the
    reference's ``Volume`` objects and returns exact ints."""
    engines[name] = dpm_moments


__all__ = [
    "ANGLES", "BenchReport", "CentralMoments3", "ENGINES", "FormatError", "InconsistencyError", "MomentTensor3",
    "Moments2D", "OpCounters", "Orientation", "ProjectionImage", "ProjectionSet", "ShapeFeatures", "Volume",
    "VolumeMeta", "apply_spacing", "brute_force_2d", "central_moments", "centroid", "count_ops", "delta",
    "dpm_moments", "dpm_moments_batch", "dpm_moments_file", "ellipsoid", "factored_moments", "feature_report",
    "load_nrrd", "load_raw", "naive_moments",
    "meta_from_header_file", "moment_indices", "normalize_scale", "project", "project_all", "project_subset",
    "random", "register", "run_bench", "shape_features", "shift_origin", "synth", "uniform", "verify_engines",
    "write_pgm", "write_raw",
]
