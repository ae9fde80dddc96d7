#!/bin/bash
# Install the UNMODIFIED reference package (/root/reference/pkg, pure Python)
# into baseline/_ref (git-ignored, travels to the GPU box with gpurun) and
# keep its own test files next to it (baseline/_ref/peakstitch_tests) so the
# reference's KATs can be run through the B200 drop-ins there
# (tests/test_reference_kats.py).  Build-container only: /root/reference does
# not exist on the GPU box.  pip resolves no dependencies (numpy / scipy /
# Pillow are in the image; --no-deps because the wheelhouse has no numpy).
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no reference at $SRC" >&2; exit 1; }
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"                      # the build writes into the tree; /root/reference is read-only
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$REPO/baseline/_ref/peakstitch_tests"
cp "$SRC/pyproject.toml" "$REPO/baseline/_ref/peakstitch_tests/reference_pyproject.toml"
rm -rf "$TMP"
echo "reference installed: $REPO/baseline/_ref"
