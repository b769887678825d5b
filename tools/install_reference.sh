#!/usr/bin/env bash
# Install the UNMODIFIED reference package (toolloop, pure Python) into
# baseline/_ref/ for bench.py's reference arm (--impl reference) and the
# CPU baseline.  baseline/_ref is git-ignored but travels to the GPU box with
# the gpurun snapshot.  The reference tree is read-only, so it is built from a
# copy under /tmp; only dependency resolution is skipped (--no-deps: click,
# fastapi, ... are already in the image and not on the timed path).
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC="${1:-/root/reference/pkg}"
TMP="$(mktemp -d)"
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
  --target "$ROOT/baseline/_ref" "$TMP/pkg"
rm -rf "$TMP"
python - "$ROOT/baseline/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import toolloop.rl.loss as L, toolloop.trajectory as T
print("reference installed:", L.__file__)
PY
