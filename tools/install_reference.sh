#!/usr/bin/env bash
# Install the UNMODIFIED reference package (topotune 0.1.0, /root/reference/pkg)
# into baseline/_ref for bench.py's reference arm (--impl reference) and the
# cpu_baseline leg.  Offline: no index, build dependencies from the image.
# /root/reference is read-only, so the build runs from a copy under /tmp.
# baseline/_ref is git-ignored but not gpurun-ignored: it travels to the box.
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -f "$SRC/pyproject.toml" ] || { echo "reference sources not found at $SRC" >&2; exit 1; }
TMP="$(mktemp -d /tmp/topotune_src.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC"/. "$TMP"/
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" "$TMP" >/dev/null
python - "$REPO/baseline/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import topotune
assert topotune.__file__.startswith(sys.argv[1]), topotune.__file__
print("installed", topotune.__file__)
PY
