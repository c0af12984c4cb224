#!/usr/bin/env bash
# Install the unmodified reference package (fpscan) as TEST / BASELINE
# INFRASTRUCTURE under baseline/_ref (git-ignored, shipped to the GPU box by
# gpurun): the bench's --impl reference arm runs its search(), and
# tests/test_reference_suite.py runs its own test files through the CUDA
# adapter (tests/reference_suite/fpscan_cuda.py). Nothing in the product
# package imports it. Run in the build container, where /root/reference exists.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference checkout at $SRC" >&2; exit 1; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"   # the build writes egg-info next to the sources; /root/reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" >/dev/null
# the reference's own test files (run against the adapter; never committed)
mkdir -p "$ROOT/baseline/_ref/fpscan_tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref/fpscan_tests/"
rm -rf "$TMP"
echo "installed fpscan into $ROOT/baseline/_ref (+ fpscan_tests/)"
