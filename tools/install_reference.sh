#!/bin/bash
# Install the UNMODIFIED reference package (ragsched) into baseline/_ref
# (git-ignored; travels to the GPU box with the snapshot).  Run in the dev
# container, where /root/reference exists.  The build writes into the source
# tree, so it installs from a copy under /tmp.
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC (not the dev container)"; exit 0; }
TMP="$(mktemp -d /tmp/ragsched_ref.XXXXXX)"
cp -r "$SRC"/. "$TMP"/
python -m pip install --quiet --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade "$TMP"
rm -rf "$TMP"
# the reference's own test suite, run on the GPU box with the drop-in active
# (tests/test_gpu_reference_sim.py); git-ignored like the install itself
rm -rf "$ROOT/baseline/_ref_tests"
cp -r "$SRC/tests" "$ROOT/baseline/_ref_tests"
echo "installed ragsched into $ROOT/baseline/_ref (tests in baseline/_ref_tests)"
