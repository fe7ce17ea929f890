#!/usr/bin/env bash
# Build the REFERENCE itself (flowplace, /root/reference/pkg) into oracle/_ref/
# -- test / baseline infrastructure only: the CPU arm of bench.py
# (--impl reference, cpu_baseline kind "reference") and golden generation.
# /root/reference is read-only, so the build runs from a copy under /tmp; the
# installed package (its Python sources + the Cython _simcore extension) lands
# in oracle/_ref/, which is git-ignored (never committed) but travels to the
# GPU box with the gpurun snapshot.  Runs only where /root/reference exists.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "build_ref: $SRC not found (reference absent): skipped"; exit 0; }
TMP="$(mktemp -d /tmp/fp_ref_build.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC"/. "$TMP"/
rm -rf "$HERE/_ref"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
    --target "$HERE/_ref" "$TMP" >/dev/null
PYTHONPATH="$HERE/_ref" FLOWPLACE_SIM_BACKEND= python - <<'PY'
import flowplace.simulate as s
name = s.backend_name()
assert name == "cython", f"reference simulator backend is {name!r}, expected cython"
print("build_ref: flowplace", s.__file__, "backend", name)
PY
