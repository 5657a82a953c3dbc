#!/usr/bin/env bash
# Installs the UNMODIFIED reference (int8flow, pure Python) into baseline/_ref
# (git-ignored, travels to the GPU box with gpurun) and places its unit suites
# next to it, for tests/test_gpu_ref_suite.py (the reference's own B=32 suites
# run against the GPU module through tests/ref_shim).  Build container only:
# /root/reference is read-only, so the wheel is built from a copy under /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
  --target "$ROOT/baseline/_ref" --upgrade "$TMP/pkg"
mkdir -p "$ROOT/baseline/_ref/int8flow_tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref/int8flow_tests/"
rm -rf "$TMP"
echo "reference installed in $ROOT/baseline/_ref"
