#!/bin/bash
# Install the reference package (the driver's reference arm and the
# reference-suite GPU test) into baseline/_ref, git-ignored but shipped to
# the GPU box by gpurun:
#   baseline/_ref/robench       pip --target install of /root/reference/pkg
#   baseline/_ref/pkg/{src,tests}  the package sources and its own test suite,
#                               run against this engine by
#                               tests/test_reference_suite_gpu.py
# /root/reference is read-only: pip builds from a copy under /tmp.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
[ -d "$SRC" ] || { echo "reference not mounted at $SRC"; exit 1; }
rm -rf /tmp/rb_refsrc "$ROOT/baseline/_ref"
cp -r "$SRC" /tmp/rb_refsrc
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --no-deps /tmp/rb_refsrc
mkdir -p "$ROOT/baseline/_ref/pkg"
cp -r "$SRC/src" "$SRC/tests" "$ROOT/baseline/_ref/pkg/"
echo "installed reference into $ROOT/baseline/_ref"
