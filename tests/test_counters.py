"""Op-count instrumentation, mirroring the reference's
complexity tests (test_moments3d.py:193-231, test_projection.py:114-119) for
the device engine's analytic tallies: the projection pass is addition-only,
P additions per voxel (P = 4 / 5 images at orders 3 / 4 -- in the moments
pipeline P - 1 images plus the profile).  Deviation: the 2D
stage multiplies every image pixel by K + 1 row powers, so multiplications
grow as n^2 (the reference's DRT route grows as n)."""
import pytest

import paper_2012_08099_b200 as vm
from paper_2012_08099_b200.projection import Orientation, project_subset

pytestmark = pytest.mark.gpu


def test_counters_zero_muls_in_projection_stage():
    v = vm.random((8, 8, 8), 8, seed=0)
    ctr = vm.OpCounters()
    project_subset(v, tuple(Orientation), ctr)
    assert ctr.multiplications == 0
    assert ctr.additions == 5 * 8 ** 3


def test_counter_dpm_additions_leading_term():
    n = 64
    v = vm.random((n, n, n), 8, seed=0)
    adds4 = vm.count_ops("dpm", v, 4).additions
    adds3 = vm.count_ops("dpm", v, 3).additions
    assert adds4 / n ** 3 == pytest.approx(5.0, rel=0.15)
    assert adds3 / n ** 3 == pytest.approx(4.0, rel=0.15)


def test_counter_dpm_multiplications_are_per_pixel():
    muls = {}
    for n in (16, 32, 64):
        v = vm.random((n, n, n), 8, seed=0)
        muls[n] = vm.count_ops("dpm", v, 4).multiplications
    # Theta(n^2): one product per image pixel and power, independent of the voxel count
    assert 3.5 < muls[32] / muls[16] < 4.5 and 3.6 < muls[64] / muls[32] < 4.4
    assert muls[64] < 64 ** 3      # far below one multiplication per voxel


def test_count_ops_matches_engine_values():
    v = vm.random((12, 9, 15), 16, seed=3)
    c = vm.OpCounters()
    t = vm.dpm_moments(v, 6, counters=c)
    assert t.values == vm.dpm_generic_moments(v, 6).values
    assert c.additions >= 7 * v.voxels.size and c.multiplications > 0
