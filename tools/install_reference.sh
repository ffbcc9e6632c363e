# Install the reference package (read-only /root/reference) into baseline/_ref
# (git-ignored; it travels to the GPU box with the snapshot), plus a copy of
# its test suite and data for the registry-swap run
# (tests/test_reference_harness.py).  Build container only.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg"
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
cp -r "$SRC/data" "$ROOT/baseline/_ref/data"
rm -rf "$TMP"
echo "installed tricount into $ROOT/baseline/_ref (+ tests, data)"
