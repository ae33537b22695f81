#!/usr/bin/env bash
# Install the UNMODIFIED reference package (`memplan`, /root/reference/pkg)
# into baseline/_ref (git-ignored, travels to the GPU box with gpurun).
# Offline: no index, no build isolation, no dependencies (numpy is in the
# image).  The reference tree is read-only, so the build runs from a copy.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC=/root/reference/pkg
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP/pkg"
rm -rf "$TMP"
PYTHONPATH="$HERE/_ref" python -c "import memplan; print('installed', memplan.__file__)"
# the reference's own test suite, run against the drop-in on the GPU box by
# tests/test_reference_suite_gpu.py (import alias tests/refsuite/memplan)
rm -rf "$HERE/_ref/reftests"
cp -r "$SRC/tests" "$HERE/_ref/reftests"
