"""The reference's own test suite (pkg/tests, 129 tests) replayed against the
``volmoments`` drop-in (volmoments/ -> this package's CUDA engine).

The suite is staged beside the reference install by
``tools/stage_reference_tests.sh`` (baseline/_ref_tests, git-ignored like
baseline/_ref); without it the test skips.  Every failure must be one of the
documented deviations below -- anything else fails.
"""
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref_tests")

# test -> why the drop-in differs (each is a documented deviation)
DEVIATIONS = {
    # the 1D-integral route (drt2d.integrals / IntegralSet / moments_1d /
    # assemble_2d, exact.*) is replaced by the device power-table kernel
    # (brute_force_2d / Moments2D, any order): the modules' tests cannot import
    "ERROR test_drt2d.py": "integral-route internals not provided",
    "ERROR test_exact.py": "volmoments.exact not provided",
    "FAILED test_moments3d.py::test_mixed_moment_formula_regression": "uses drt2d.assemble_2d(integrals(...))",
    # Python seams the reference's fault-injection tests monkeypatch do not
    # exist: the placement / cross-axis solve runs in the device epilogue
    "FAILED test_harness.py::test_verify_names_divergent_index_on_fault": "no moments3d._cross_axis_moments seam",
    "FAILED test_harness.py::test_cli_verify_fault_names_index": "no moments3d._cross_axis_moments seam",
    "FAILED test_moments3d.py::test_cross_axis_helper_is_live": "no moments3d._cross_axis_moments seam",
    "FAILED test_moments3d.py::test_inconsistency_error_on_disagreeing_routes": "no moments3d.project_subset seam",
    # extension: orders 5 and 6 are accepted (BASELINE config 5 needs order 6)
    "FAILED test_moments3d.py::test_order_validation": "order 5 accepted",
    # the device 2D stage multiplies every image pixel by its row powers:
    # Theta(n^2) multiplications instead of the integral route's Theta(n)
    "FAILED test_moments3d.py::test_counter_scaling_dpm_is_linear": "Theta(n^2) multiplications",
}


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="reference suite not staged (tools/stage_reference_tests.sh)")
def test_reference_suite_against_the_dropin():
    env = dict(os.environ, PYTHONPATH=ROOT)
    proc = subprocess.run([sys.executable, "-m", "pytest", ".", "-q", "-p", "no:cacheprovider", "-rfE",
                           "--continue-on-collection-errors", "--tb=no"],
                          cwd=SUITE, env=env, capture_output=True, text=True, timeout=1800)
    out = proc.stdout
    bad = set()
    for line in out.splitlines():
        m = re.match(r"^(FAILED|ERROR) (\S+)", line)
        if m:
            bad.add(f"{m.group(1)} {m.group(2)}")
    unexpected = sorted(bad - set(DEVIATIONS))
    assert not unexpected, "reference tests failing beyond the documented deviations:\n" + "\n".join(unexpected)
    m = re.search(r"(\d+) passed", out)
    assert m and int(m.group(1)) >= 97, out[-2000:]
    import volmoments
    assert volmoments.dpm_moments.__module__ == "paper_2012_08099_b200.moments3d"


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="reference suite not staged")
def test_deviation_list_is_current():
    """No documented deviation may silently start passing (keep the list honest)."""
    env = dict(os.environ, PYTHONPATH=ROOT)
    proc = subprocess.run([sys.executable, "-m", "pytest", ".", "-q", "-p", "no:cacheprovider", "-rfE",
                           "--continue-on-collection-errors", "--tb=no"],
                          cwd=SUITE, env=env, capture_output=True, text=True, timeout=1800)
    bad = {f"{m.group(1)} {m.group(2)}" for m in re.finditer(r"^(FAILED|ERROR) (\S+)", proc.stdout, re.M)}
    assert set(DEVIATIONS) <= bad, sorted(set(DEVIATIONS) - bad)
