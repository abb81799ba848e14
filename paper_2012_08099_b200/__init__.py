"""B200-native Discrete Projection Moment (DPM) hot path.

A drop-in for the hot path of the reference package ``volmoments``
(arXiv 2012.08099): the same public names for volumes, projections and 3D
moments, with every stage running in hand-written sm_100a CUDA kernels behind
the C ABI in include/dpm_b200.h.  There is no CPU fallback: without the CUDA
library (paper_2012_08099_b200/libdpm_b200.so) and a GPU, compute calls raise.
"""
from . import drt2d, harness
from .harness import BenchReport, run_bench, verify_engines
from .counters import OpCounters
from .drt2d import Moments2D, brute_force_2d, image_moments, shift_origin
from .errors import FormatError, InconsistencyError
from .features import (CentralMoments3, ShapeFeatures, apply_spacing, central_moments, centroid, feature_report,
                       normalize_scale, shape_features)
from .moments3d import (ENGINES, MomentTensor3, count_ops, dpm_generic_moments, dpm_moments, dpm_moments_batch,
                        dpm_moments_file, factored_moments, moment_indices, naive_moments)
from .projection import (ANGLES, Orientation, ProjectionImage, ProjectionSet, project, project_all,
                         project_extended, project_subset, write_pgm)
from .volio import VolumeMeta, load_nrrd, load_raw, meta_from_header_file, open_nrrd, open_raw, write_raw
from .volume import Volume, delta, ellipsoid, random, synth, uniform

__version__ = "0.1.0"

__all__ = [
    "ANGLES", "BenchReport", "CentralMoments3", "ENGINES", "FormatError", "ShapeFeatures", "apply_spacing", "central_moments",
    "centroid", "feature_report", "normalize_scale", "shape_features", "InconsistencyError", "Moments2D", "MomentTensor3", "OpCounters",
    "Orientation", "ProjectionImage", "ProjectionSet", "Volume", "count_ops", "delta",
    "VolumeMeta", "brute_force_2d", "dpm_generic_moments", "factored_moments", "naive_moments", "dpm_moments", "dpm_moments_batch", "harness", "run_bench", "synth", "verify_engines", "dpm_moments_file", "drt2d",
    "ellipsoid", "image_moments", "load_nrrd", "load_raw", "meta_from_header_file", "open_nrrd", "open_raw",
    "moment_indices", "project", "project_all",
    "project_extended", "project_subset", "random", "shift_origin", "uniform", "write_pgm", "write_raw",
]
