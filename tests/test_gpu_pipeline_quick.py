"""Quick end-to-end parity of the CUDA pipeline against the C oracle."""
import numpy as np
import pytest

import oracle
import paper_2012_08099_b200 as vm

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,bits,order", [((5, 4, 3), 8, 3), ((7, 6, 5), 16, 4), ((9, 7, 5), 8, 6),
                                               ((64, 64, 64), 8, 3), ((33, 17, 20), 16, 6)])
def test_dpm_matches_oracle(cuda, dims, bits, order):
    v = vm.random(dims, bits, seed=3)
    got = vm.dpm_moments(v, order)
    want = oracle.naive(v.voxels, order)
    assert got.values == want


@pytest.mark.parametrize("dims", [(1, 1, 1), (5, 3, 2), (16, 16, 16), (70, 9, 33)])
def test_projections_match_oracle(cuda, dims):
    v = vm.random(dims, 16, seed=1)
    got = vm.project_extended(v)
    want = oracle.project(v.voxels, 7)
    for k, name in enumerate(vm.projection.EXTENDED_NAMES):
        assert np.array_equal(got[name].pixels, want[k]), name
