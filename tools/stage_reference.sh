#!/usr/bin/env bash
# Install the UNMODIFIED reference (embedview) into baseline/_ref (git-ignored,
# travels to the GPU box with the gpurun snapshot) and stage its own test
# suite beside it, so tests/test_gpu_dropin.py can run the reference's tests
# through esom.install() on the B200.  Run here (the container that has
# /root/reference); nothing under baseline/_ref is committed.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
REF=/root/reference/pkg
[ -d "$REF" ] || { echo "no reference at $REF"; exit 1; }
TMP=$(mktemp -d)
cp -r "$REF" "$TMP/pkg"   # the build writes into its source tree; /root/reference is read-only
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade "$TMP/pkg" > /dev/null
rm -rf "$ROOT/baseline/_ref/embedview_tests"
cp -r "$REF/tests" "$ROOT/baseline/_ref/embedview_tests"
rm -rf "$TMP"
echo "staged: $(ls "$ROOT/baseline/_ref")"
