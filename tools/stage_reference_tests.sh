#!/bin/bash
# Stage the reference's own test suite beside the driver's reference install
# (baseline/_ref_tests, git-ignored like baseline/_ref: it travels to the GPU
# box with gpurun, never into history) so tests/test_gpu_reference_suite.py can
# replay it against the `volmoments` drop-in.  Run in the build container.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=/root/reference/pkg/tests
[ -d "$SRC" ] || { echo "no $SRC"; exit 1; }
rm -rf "$ROOT/baseline/_ref_tests"
mkdir -p "$ROOT/baseline/_ref_tests"
cp "$SRC"/*.py "$ROOT/baseline/_ref_tests/"
echo "staged $(ls "$ROOT/baseline/_ref_tests" | wc -l) files into baseline/_ref_tests"
