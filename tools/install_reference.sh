#!/bin/bash
# Installs the UNMODIFIED reference package (limapper, /root/reference/pkg) into baseline/_ref
# (git-ignored; it travels to the GPU box with gpurun) and copies its own pytest suite next to
# it (baseline/_ref/limapper_tests), so tests/test_gpu_reference_suite.py can run the
# reference's tests against the drop-in (integrate.patch) on the B200.  Needs /root/reference,
# i.e. runs in the build container, not on the GPU box.
set -e
cd "$(dirname "$0")/.."
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC here (the GPU box has only the installed copy)"; exit 0; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"          # the build writes egg-info into the source tree
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref --upgrade "$TMP/pkg" > "$TMP/pip.log" 2>&1 || { cat "$TMP/pip.log"; exit 1; }
rm -rf baseline/_ref/limapper_tests
cp -r "$SRC/tests" baseline/_ref/limapper_tests
rm -rf "$TMP"
python - <<'PY'
import sys
sys.path.insert(0, "baseline/_ref")
import limapper, limapper.registration
print("installed", limapper.__file__)
PY
