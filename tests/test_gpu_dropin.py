"""The ``volmoments`` drop-in name and the reference-side engine registration
(INTEGRATION.md §2): the CUDA engine added to the REFERENCE's own ENGINES and
cross-checked by the reference's own harness.verify_engines against its CPU
engines (naive, factored, dpm), on reference Volume objects."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_volmoments_name_resolves_to_the_cuda_engine():
    import volmoments as vm
    import volmoments.moments3d as m3
    from volmoments.projection import project_subset  # noqa: F401  (reference import paths)
    assert set(m3.ENGINES) >= {"naive", "factored", "dpm"}
    v = vm.random((9, 7, 5), 16, seed=3)
    t = vm.dpm_moments(v, 4)
    assert t.values == vm.naive_moments(v, 4).values == vm.factored_moments(v, 4).values


def test_cuda_engine_registered_in_the_reference_registry():
    from oracle import reference
    ref = reference.load()
    if ref is None:
        pytest.skip("reference install (baseline/_ref) not on this host")
    import importlib

    import volmoments
    m3 = importlib.import_module("volmoments_ref.moments3d")
    harness = importlib.import_module("volmoments_ref.harness")
    volmoments.register(m3.ENGINES)
    try:
        assert "dpm_cuda" in m3.ENGINES
        res = harness.verify_engines((17, 13, 11), seeds=3, orders=(3, 4))
        assert res.ok, res
        v = ref.random((40, 30, 20), 16, seed=5)
        assert m3.ENGINES["dpm_cuda"](v, 4).values == m3.ENGINES["naive"](v, 4).values
    finally:
        m3.ENGINES.pop("dpm_cuda", None)
