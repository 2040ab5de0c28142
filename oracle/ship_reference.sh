#!/usr/bin/env bash
# Install the UNMODIFIED reference package (annq, pure Python) untracked under
# baseline/_ref so it travels to the GPU box with the repo snapshot:
#   * bench.py --impl reference times annq.encode_dataset from it;
#   * tests/test_gpu_reference_suite.py runs the reference's own unit tests
#     (copied next to it, baseline/_ref/annq_tests) with install() patched in.
# baseline/_ref is git-ignored (never committed).  Needs /root/reference, so it
# runs in the build container only; a box without baseline/_ref skips those legs.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${REFERENCE_ROOT:-/root/reference}/pkg"
[ -d "$SRC/src/annq" ] || { echo "no reference at $SRC; nothing to ship"; exit 0; }
DEST="$ROOT/baseline/_ref"
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"                    # the reference tree is read-only
rm -rf "$DEST"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$DEST" "$TMP/pkg"
mkdir -p "$DEST/annq_tests"
cp "$SRC"/tests/*.py "$DEST/annq_tests/"
echo "reference installed at $DEST ($(ls "$DEST/annq_tests" | wc -l) test files)"
