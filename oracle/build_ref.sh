#!/usr/bin/env bash
# Test infrastructure only (see oracle/README.md): builds the UNMODIFIED
# reference package `anchorqp` (Cython backend) from /root/reference/pkg into
# oracle/_ref/ so the parity tests, the golden-fixture generator and the
# bench reference arm can import the real reference.  /root/reference is
# read-only, so the build runs from a scratch copy under /tmp.  Outputs land
# only in oracle/_ref/ (git-ignored; it still ships to the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${AQP_REFERENCE_PKG:-/root/reference/pkg}"
if [ ! -d "$SRC" ]; then
  echo "reference package not found at $SRC; skipping oracle/_ref build" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/aqp_refbuild.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --target "$HERE/_ref" "$TMP/pkg"
# the reference's own tests, for oracle/ref_suite_plugin.py (git-ignored with the rest of _ref)
cp -r "$TMP/pkg/tests" "$HERE/_ref/tests"
PYTHONPATH="$HERE/_ref" python -c "import anchorqp; b = anchorqp.active_backend(); assert b == 'cython', b; print('oracle/_ref: anchorqp', anchorqp.__version__, 'backend', b)"
