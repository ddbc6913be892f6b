#!/bin/bash
# Install the UNMODIFIED reference package (`bitserial`, pure Python) into baseline/_ref/ so
# bench.py --impl reference and the cpu_baseline leg time the reference's own code path
# (oracle/ref_baseline.py).  Offline: no index, no dependency resolution (numpy is in the
# image; jsonschema too).  The source tree is read-only, so build from a copy under /tmp.
# baseline/_ref/ is git-ignored but travels to the GPU box with the gpurun snapshot.
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d /tmp/bitserial_src.XXXXXX)
cp -r "$SRC"/. "$TMP"/
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP"
rm -rf "$TMP"
PYTHONPATH="$ROOT/baseline/_ref" python -c "import bitserial; print('installed', bitserial.__file__)"
