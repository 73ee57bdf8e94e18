#!/usr/bin/env bash
# Pod-local install of the reference package into baseline/_ref (git-ignored,
# not gpurun-ignored: it travels to the GPU box with the snapshot).  The one
# offline install the task allows; the reference's own tests are copied beside
# it for tests/test_reference_suite.py (they are not part of its wheel).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"            # the build writes into its source tree; /root/reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
mkdir -p "$ROOT/baseline/_ref/tests"
cp "$TMP/pkg/tests/"*.py "$ROOT/baseline/_ref/tests/"
rm -rf "$TMP"
echo "reference installed in $ROOT/baseline/_ref (tests in baseline/_ref/tests)"
