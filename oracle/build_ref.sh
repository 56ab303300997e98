#!/usr/bin/env bash
# Install the reference package (pure Python + numba; /root/reference/pkg) into
# oracle/_ref/ -- the CPU baseline of record that bench.py times (oracle/ref_runner.py).
# Offline, no dependency resolution (numpy / numba / pyyaml are in the image);
# installed from a /tmp copy because the setuptools build writes into the
# source tree and /root/reference is read-only.  oracle/_ref/ is git-ignored
# (not gpurun-ignored, so it travels to the GPU box).  Never copies reference
# sources into the repository history.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
SRC="${1:-/root/reference/pkg}"
if [ ! -f "$SRC/pyproject.toml" ]; then
  echo "build_ref: no reference at $SRC (skipped)"; exit 0
fi
TMP="$(mktemp -d /tmp/rgb_refbuild.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg"
echo "build_ref: installed $(ls "$HERE/_ref" | tr '\n' ' ')"
