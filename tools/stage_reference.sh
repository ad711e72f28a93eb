#!/bin/bash
# Stage the UNMODIFIED reference package (romtopt) and its own test-suite under baseline/_ref
# (git-ignored; travels to the GPU box with the gpurun snapshot).  Used by bench.py's CPU arms
# (romtopt itself where it can run) and by tests/test_gpu_dropin.py (the reference's tests and
# TrustRegionDriver run against the B200 drop-in classes).  Needs /root/reference (this build
# container only); the install is offline (--no-index), from a copy (the source tree is read-only).
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP/pkg"
mkdir -p "$REPO/baseline/_ref/romtopt_tests"
cp "$SRC"/tests/*.py "$REPO/baseline/_ref/romtopt_tests/"
# the reference's own cached MMA reference histories (mbb, cantilever, mbb-small), read by its
# acceptance suite from <tests>/../.ref_cache
if [ -d "$SRC/.ref_cache" ]; then cp -r "$SRC/.ref_cache" "$REPO/baseline/_ref/.ref_cache"; chmod -R u+w "$REPO/baseline/_ref/.ref_cache"; fi
rm -rf "$TMP"
echo "staged romtopt + tests in $REPO/baseline/_ref"
