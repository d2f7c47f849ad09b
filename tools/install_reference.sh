#!/bin/bash
# Offline install of the reference package (pure Python "evsim") into the
# git-ignored baseline/_ref (it travels to the GPU box with gpurun; it is not
# product code and nothing in the package imports it):
#   * baseline/_ref/evsim           -- the unmodified reference, pip-installed from a /tmp copy
#   * baseline/_ref/pkg_tests/{tests,configs,golden}
#                                   -- the reference's own test suite and the files it opens,
#                                      run against the drop-in by tests/test_gpu_reference_suite.py
# Used by bench.py --impl reference (the reference's own CPU path) as well.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference at $SRC"; exit 1; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" > "$TMP/pip.log" 2>&1 || { tail -5 "$TMP/pip.log"; exit 1; }
mkdir -p "$ROOT/baseline/_ref/pkg_tests"
cp -r "$SRC/tests" "$SRC/configs" "$SRC/golden" "$ROOT/baseline/_ref/pkg_tests/"
rm -rf "$TMP"
echo "installed: $(ls "$ROOT/baseline/_ref")"
