#!/bin/sh
# Install the UNMODIFIED reference package (kvweaver, /root/reference/pkg) into
# baseline/_ref — git-ignored, but it travels to the GPU box with the gpurun
# snapshot — together with the reference's own test files (baseline/_ref/
# kvweaver_tests).  Uses: bench.py --impl reference (the reference CPU toy at
# configs[0]) and tests/test_reference_unmodified.py (the reference's suites
# and test files run against this package through an import alias).
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"  # the build writes into the source tree; /root/reference is read-only
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref/kvweaver_tests"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/kvweaver_tests"
rm -rf "$TMP"
echo "reference installed in $ROOT/baseline/_ref"
