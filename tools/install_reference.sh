#!/usr/bin/env bash
# Install the UNMODIFIED reference (epivec) into baseline/_ref/ (git-ignored,
# shipped to the GPU box with the gpurun snapshot), plus a copy of its own
# test suite under baseline/_ref/tests/ so `tests/test_gpu_reference_suite.py`
# can run it against GpuEngine there.  /root/reference is read-only: the
# build happens from a copy under /tmp.  Run from the repo root, in this
# container (the GPU box has no /root/reference).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
DST="$ROOT/baseline/_ref"
TMP="$(mktemp -d /tmp/epivec_src.XXXXXX)"
cp -r "$SRC/." "$TMP/"
rm -rf "$DST"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$DST" "$TMP" >/dev/null
rm -rf "$DST/tests"
cp -r "$SRC/tests" "$DST/tests"
cp "$SRC/pyproject.toml" "$DST/tests/pyproject.toml.ref"
rm -rf "$TMP"
echo "installed epivec into $DST ($(ls "$DST/tests" | wc -l) test files)"
