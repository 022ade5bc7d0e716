#!/usr/bin/env bash
# Build the UNMODIFIED reference package (rlra 0.1.0, Python + one Cython GEPP
# kernel) from /root/reference/pkg into oracle/_ref/ so that tests and the
# bench's reference arm can import it.  Test infrastructure only: nothing in
# the product package imports oracle/.
#
# Recipe: copy pkg/ to a scratch dir (the mount is
# read-only), drop the shipped Cython-3.2.8-generated _lu_cython.c so the
# local Cython regenerates it, then pip-install offline into oracle/_ref.
# oracle/_ref/ is git-ignored but travels to the GPU box with gpurun.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${RLRA_REFERENCE:-/root/reference}/pkg"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "reference not present at $SRC; keeping prebuilt $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/rlra_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -f "$TMP/pkg/src/rlra/_lu_cython.c"
rm -rf "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --target "$OUT" "$TMP/pkg"
# the reference's own test files, next to the build (git-ignored, not
# committed): tests/test_reference_suite_gpu.py runs them against the B200
# backend and the aliased hot path on the GPU box, where /root/reference is absent
cp -r "$SRC/tests" "$OUT/tests"
python - "$OUT" <<'PY'
import os, sys
sys.path.insert(0, sys.argv[1])
os.environ["RLRA_BACKEND"] = "compiled"
import rlra
assert rlra.BACKEND == "compiled", rlra.BACKEND
print("oracle/_ref: rlra", rlra.__version__, "backend", rlra.BACKEND)
PY
