"""ctypes binding of the C ABI in include/dpm_b200.h (libdpm_b200.so).

This is the reference-facing plugin boundary: the reference package is pure
Python, so its natural foreign-function binding is ctypes.  Nothing here
computes; every entry point enqueues CUDA work on a caller-supplied stream.
A missing or unloadable library raises immediately -- there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os
from functools import lru_cache

_HERE = os.path.dirname(os.path.abspath(__file__))
# DPM_LIB_PATH overrides the in-tree library (A/B builds of kernel variants only)
LIB_PATH = os.environ.get("DPM_LIB_PATH") or os.path.join(_HERE, "libdpm_b200.so")

DPM_OK, DPM_EINVAL, DPM_EOVERFLOW, DPM_ECUDA, DPM_EWORKSPACE = 0, 1, 2, 3, 4
DPM_ST_DISAGREE, DPM_ST_NONEXACT, DPM_ST_MASS = 1, 2, 4
DPM_U8, DPM_U16, DPM_I16 = 1, 2, 3
MAX_IMAGES, MAX_ORDER = 7, 6
DPM_ACC_IMAGES, DPM_ACC_PROFILE, DPM_ACC_PROFILE_T = 0, 1, 2

#: every symbol include/dpm_b200.h declares (checked by tests/test_capi_symbols.py)
EXPORTS = (
    "dpm_num_images", "dpm_num_moments3d", "dpm_num_moments2d", "dpm_image_layout",
    "dpm_project_workspace_bytes", "dpm_project", "dpm_moments2d", "dpm_derive3d",
    "dpm_workspace_bytes", "dpm_moments", "dpm_check_envelope", "dpm_acc_add",
    "dpm_synth_noise_u16", "dpm_last_launch_count", "dpm_strerror", "dpm_image_moments2d",
    "dpm_project_generic", "dpm_profile_layout", "dpm_project_profile", "dpm_zero_profile_buffers",
    "dpm_project_profile_zeroed", "dpm_moments2d_profile",
    "dpm_partial_workspace_bytes", "dpm_moments_partial", "dpm_moments2d_profile_derive",
    "dpm_moments_acc_kind", "dpm_moments_image_layout", "dpm_direct_workspace_bytes", "dpm_direct_moments",
)
DPM_DIRECT_NAIVE, DPM_DIRECT_FACTORED = 0, 1


class VolumeDesc(ctypes.Structure):
    """Mirror of ``dpm_volume_desc``."""
    _fields_ = [
        ("L", ctypes.c_int64), ("M", ctypes.c_int64), ("N", ctypes.c_int64),
        ("B", ctypes.c_int64),
        ("stride_y", ctypes.c_int64), ("stride_z", ctypes.c_int64), ("stride_b", ctypes.c_int64),
        ("dtype", ctypes.c_int32), ("offset", ctypes.c_int32),
        ("z0", ctypes.c_int64),
    ]


class NativeError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {strerror(code)} (code {code})")


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"CUDA extension {LIB_PATH} is missing: build it with "
            f"`python -c 'import __graft_entry__ as g; g.build()'` (make -C paper_2012_08099_b200/csrc)")
    L = ctypes.CDLL(LIB_PATH)
    i64, i32, vp, sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_size_t
    pdesc = ctypes.POINTER(VolumeDesc)
    sig = {
        "dpm_num_images": (ctypes.c_int, [ctypes.c_int]),
        "dpm_num_moments3d": (ctypes.c_int, [ctypes.c_int]),
        "dpm_num_moments2d": (ctypes.c_int, [ctypes.c_int]),
        "dpm_image_layout": (ctypes.c_int, [pdesc, ctypes.c_int] + [ctypes.POINTER(i64)] * 4),
        "dpm_moments_image_layout": (ctypes.c_int, [pdesc, ctypes.c_int, ctypes.c_int] + [ctypes.POINTER(i64)] * 4),
        "dpm_moments_acc_kind": (ctypes.c_int, [pdesc, ctypes.c_int]),
        "dpm_direct_workspace_bytes": (sz, [pdesc, ctypes.c_int]),
        "dpm_direct_moments": (ctypes.c_int, [pdesc, vp, ctypes.c_int, ctypes.c_int, vp, sz, vp, vp, vp]),
        "dpm_project_workspace_bytes": (sz, [pdesc, ctypes.c_int]),
        "dpm_project": (ctypes.c_int, [pdesc, vp, ctypes.c_int, ctypes.POINTER(vp), vp, sz, vp]),
        "dpm_project_generic": (ctypes.c_int, [pdesc, vp, ctypes.c_int, ctypes.POINTER(vp), vp]),
        "dpm_moments2d": (ctypes.c_int, [pdesc, ctypes.c_int, ctypes.POINTER(vp), ctypes.c_int, vp, vp]),
        "dpm_derive3d": (ctypes.c_int, [pdesc, vp, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp]),
        "dpm_profile_layout": (ctypes.c_int, [pdesc, ctypes.c_int, ctypes.POINTER(i64), ctypes.POINTER(i64),
                                              ctypes.POINTER(ctypes.c_int)]),
        "dpm_project_profile": (ctypes.c_int, [pdesc, vp, ctypes.c_int, ctypes.POINTER(vp), vp, vp]),
        "dpm_zero_profile_buffers": (ctypes.c_int, [pdesc, ctypes.c_int, ctypes.POINTER(vp), vp, vp]),
        "dpm_project_profile_zeroed": (ctypes.c_int, [pdesc, vp, ctypes.c_int, ctypes.POINTER(vp), vp, vp]),
        "dpm_moments2d_profile": (ctypes.c_int, [pdesc, ctypes.c_int, ctypes.POINTER(vp), vp, vp, vp]),
        "dpm_moments2d_profile_derive": (ctypes.c_int, [pdesc, ctypes.c_int, ctypes.POINTER(vp), vp, vp, vp, vp, vp,
                                                         vp, vp]),
        "dpm_partial_workspace_bytes": (sz, [pdesc, ctypes.c_int]),
        "dpm_moments_partial": (ctypes.c_int, [pdesc, vp, ctypes.c_int, vp, sz, vp, vp]),
        "dpm_image_moments2d": (ctypes.c_int, [vp, i64, i64, i64, i64, ctypes.c_int, vp, vp]),
        "dpm_workspace_bytes": (sz, [pdesc, ctypes.c_int]),
        "dpm_moments": (ctypes.c_int, [pdesc, vp, ctypes.c_int, vp, sz, vp, vp, vp, vp]),
        "dpm_check_envelope": (ctypes.c_int, [i64, i64, i64, i64, ctypes.c_int]),
        "dpm_acc_add": (ctypes.c_int, [vp, vp, i64, vp]),
        "dpm_synth_noise_u16": (ctypes.c_int, [vp, i64, i64, i64, i64, ctypes.c_uint64, vp]),
        "dpm_last_launch_count": (ctypes.c_int, []),
        "dpm_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _ = i32
    return L


def strerror(code: int) -> str:
    return lib().dpm_strerror(int(code)).decode()


def check(code: int, where: str) -> None:
    """Map a C-ABI status to the reference's exception taxonomy."""
    if code == DPM_OK:
        return
    if code == DPM_EINVAL:
        raise ValueError(f"{where}: {strerror(code)}")
    if code == DPM_EOVERFLOW:
        raise OverflowError(f"{where}: {strerror(code)}")
    raise NativeError(code, where)


def last_launch_count() -> int:
    return int(lib().dpm_last_launch_count())
