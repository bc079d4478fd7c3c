#!/bin/bash
# Test infrastructure: install the UNMODIFIED reference package (pure
# Python, /root/reference/pkg) into oracle/_ref so the reference arm of
# bench.py (--impl reference) and the CPU baseline can run the reference
# itself on the GPU box, where /root/reference does not exist.  oracle/_ref
# is git-ignored (not product source) but travels with gpurun snapshots.
# Offline: no index, no dependencies (numpy is in the image; matplotlib is
# only used by the reference's figures module).
set -euo pipefail
here="$(cd "$(dirname "$0")" && pwd)"
src=/root/reference/pkg
[ -d "$src" ] || { echo "vendor_ref: $src not present (GPU box?): keeping oracle/_ref as is"; exit 0; }
tmp="$(mktemp -d)"
trap 'rm -rf "$tmp"' EXIT
cp -r "$src" "$tmp/pkg"          # the build writes egg-info: never into /root/reference
rm -rf "$here/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --find-links /opt/wheelhouse --target "$here/_ref" "$tmp/pkg"
python - "$here/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import specpipe
print("vendor_ref: specpipe", specpipe.__version__, "->", sys.argv[1])
PY
