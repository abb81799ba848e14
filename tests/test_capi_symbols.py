"""The C-ABI library loads (no GPU needed) and exports exactly what include/dpm_b200.h declares."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
from paper_2012_08099_b200 import _native as nat

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "dpm_b200.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"DPM_API\s+[\w\s\*]+?\b(dpm_\w+)\s*\(", txt)))


def test_header_declares_the_exported_list():
    assert declared() == sorted(nat.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = nat.lib()
    for name in declared():
        assert getattr(lib, name) is not None, name


def test_host_only_entry_points():
    lib = nat.lib()
    assert [lib.dpm_num_images(k) for k in (3, 4, 5, 6)] == [4, 5, 6, 7]
    assert lib.dpm_num_images(2) == 0 and lib.dpm_num_images(7) == 0
    assert [lib.dpm_num_moments3d(k) for k in (3, 4, 6)] == [20, 35, 84]
    assert lib.dpm_strerror(nat.DPM_EINVAL).decode() == "invalid argument"
    assert lib.dpm_check_envelope(2048, 2048, 2048, 65535, 6) == nat.DPM_OK
    assert lib.dpm_check_envelope(65536, 65536, 65536, 65535, 6) == nat.DPM_EOVERFLOW
    assert lib.dpm_check_envelope(0, 1, 1, 1, 3) == nat.DPM_EINVAL


@pytest.mark.parametrize("dims,z0", [((5, 3, 2), 0), ((512, 512, 230), 0), ((7, 9, 11), 13), ((2048, 2048, 256), 1024)])
def test_image_layout_matches_oracle(dims, z0):
    d = nat.VolumeDesc()
    d.L, d.M, d.N = dims
    d.B = 1
    d.z0 = z0
    for img in range(7):
        out = [ctypes.c_int64() for _ in range(4)]
        assert nat.lib().dpm_image_layout(ctypes.byref(d), img, *[ctypes.byref(o) for o in out]) == 0
        assert tuple(o.value for o in out) == oracle.layout(dims, img, z0)


def test_invalid_arguments_rejected_without_a_device():
    d = nat.VolumeDesc()
    d.L = d.M = d.N = 4
    d.B = 1
    d.stride_y, d.stride_z, d.stride_b = 4, 16, 64
    d.dtype = 9   # unsupported dtype
    imgs = (ctypes.c_void_p * 4)()
    assert nat.lib().dpm_project(ctypes.byref(d), None, 4, imgs, None, 0, None) == nat.DPM_EINVAL
    d.dtype = nat.DPM_U16
    d.L = 70000   # longest ray * 65535 would overflow a uint32 ray sum
    d.stride_y, d.stride_z = 70000, 280000
    assert nat.lib().dpm_project(ctypes.byref(d), None, 4, imgs, None, 0, None) == nat.DPM_EOVERFLOW
    with pytest.raises(ValueError):
        nat.check(nat.DPM_EINVAL, "x")
    with pytest.raises(OverflowError):
        nat.check(nat.DPM_EOVERFLOW, "x")
    assert np.int64  # numpy import used


def test_envelope_order6_profile_rule():
    """Order 6 adds mass * max(L,M,N)^6 < 2^116 (the profile solve)
    on top of the 2^126 image envelope: this shape passes the latter, not the former."""
    lib = nat.lib()
    n = 4096
    assert lib.dpm_check_envelope(n, n, n, 257, 5) == nat.DPM_OK        # images + profile solve fine at order 5
    assert lib.dpm_check_envelope(n, n, n, 257, 6) == nat.DPM_EOVERFLOW
    assert lib.dpm_check_envelope(n, n, n, 255, 6) == nat.DPM_OK        # just below 2^116


def _desc(dims, z0=0, dtype=nat.DPM_U16):
    d = nat.VolumeDesc()
    d.L, d.M, d.N = dims
    d.B = 1
    d.stride_y, d.stride_z, d.stride_b = dims[0], dims[0] * dims[1], dims[0] * dims[1] * dims[2]
    d.dtype = dtype
    d.z0 = z0
    return d


@pytest.mark.parametrize("dims,z0", [((2048, 2048, 256), 1024), ((256, 40, 24), 0), ((264, 9, 150), 17),
                                     ((203, 11, 13), 0), ((128, 128, 128), 0), ((64, 64, 64), 5)])
@pytest.mark.parametrize("order", [3, 4, 5, 6])
def test_moments_layout_geometry(dims, z0, order):
    """The moments pipeline's image geometry: classic for narrow volumes, layout
    T (x and z exchanged, slab offset on the x' axis) for L >= 192."""
    lib = nat.lib()
    d = _desc(dims, z0)
    L, M, N = dims
    kind = lib.dpm_moments_acc_kind(ctypes.byref(d), order)
    wide = L >= 192
    assert kind == (nat.DPM_ACC_PROFILE_T if wide else nat.DPM_ACC_PROFILE)
    for img in range(4 if order <= 3 else order + 1):
        out = [ctypes.c_int64() for _ in range(4)]
        rc = lib.dpm_moments_image_layout(ctypes.byref(d), order, img, *[ctypes.byref(o) for o in out])
        if img == 2:
            assert rc == nat.DPM_EINVAL
            continue
        assert rc == 0
        got = tuple(o.value for o in out)
        if not wide:
            assert got == oracle.layout(dims, img, z0)
        else:
            W, H, ai, aj = oracle.layout((N, M, L), img, 0)    # the transposed volume at z0 = 0
            shift = z0 if img == 0 or img >= 3 else 0          # indices containing x' = z carry the slab offset
            assert got == (W, H, ai + shift, aj)
    wq, ai, t = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int()
    assert lib.dpm_profile_layout(ctypes.byref(d), order, ctypes.byref(wq), ctypes.byref(ai), ctypes.byref(t)) == 0
    at = abs(t.value)
    if wide:
        assert wq.value == N + at * (L - 1)
        assert ai.value == (0 if t.value > 0 else -at * (L - 1)) + z0
    else:
        assert wq.value == L + at * (N - 1)
