#!/bin/sh
# Test infrastructure (not product code): install the UNMODIFIED reference
# package `psdcone` (pure Python over numpy) from /root/reference/pkg into
# oracle/_ref/ with an offline pip install, so that the GPU box — which has no
# /root/reference — can (a) drive the reference's own public API through
# paper_2410_19208_b200.install() in `pytest -m gpu` (tests/test_gpu_dropin.py)
# and (b) time the real psdcone.ran_proj as bench.py's reference arm.
#
# oracle/_ref/ is git-ignored (no reference source enters history) and NOT
# gpurun-ignored, so it travels with the snapshot like the built .so files.
# The build is done from a copy under /tmp because setuptools writes
# build/ and *.egg-info/ next to the sources and /root/reference is read-only.
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=${1:-/root/reference/pkg}
if [ ! -f "$SRC/pyproject.toml" ]; then
  echo "make_ref.sh: $SRC not present; keeping the existing oracle/_ref (if any)"
  exit 0
fi
TMP=$(mktemp -d /tmp/psdcone_ref.XXXXXX)
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref.tmp"
${PYTHON:-python} -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$HERE/_ref.tmp" "$TMP/pkg"
rm -rf "$HERE/_ref"
mv "$HERE/_ref.tmp" "$HERE/_ref"
echo "make_ref.sh: installed psdcone into $HERE/_ref"
