#!/usr/bin/env bash
# Install the unmodified reference package (`dimreal`, /root/reference/pkg) into
# baseline/_ref for bench.py's reference arm.  Offline: the image's wheelhouse only; the
# reference's own dependencies (numpy, scipy, numba, cv2, torch) are already in the image,
# so dependency resolution is skipped (--no-deps).  The build writes into its source
# tree, so it runs from a copy under /tmp (/root/reference is read-only).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d /tmp/dimreal_src.XXXXXX)"
cp -r "$SRC"/. "$TMP"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$HERE/_ref" "$TMP"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$HERE/_ref'); import dimreal.inpaint.dstt as d; print('dimreal installed:', d.__file__)"
