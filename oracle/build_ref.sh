#!/usr/bin/env bash
# Installs the UNMODIFIED reference package (/root/reference/pkg, pure Python + numpy) into
# oracle/_ref for the bench's reference arm (oracle/ref_step.py).  oracle/_ref is git-ignored
# (never committed) but not gpurun-ignored, so it travels to the GPU box, where
# /root/reference does not exist.  The reference's build writes into its source tree, so it
# is installed from a scratch copy (/root/reference is read-only).  No network: --no-index.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${REFERENCE_PKG:-/root/reference/pkg}"
[ -d "$SRC" ] || { echo "no reference at $SRC; keeping existing oracle/_ref" >&2; exit 0; }
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --target "$HERE/_ref" "$TMP/pkg"
python - "$HERE/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import composer
print("oracle/_ref: composer", composer.__file__)
PY
