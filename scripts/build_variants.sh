#!/bin/bash
# Build a tuning variant of libclaw.so into build/variants/libclaw_NAME.so with
# extra -D knobs (same sources and split as build.py), e.g.
#   scripts/build_variants.sh w24 -DCLAW_RES_WARPS=24
# then run with CLAW_LIB=build/variants/libclaw_w24.so.
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/variants
python - "$name" "$@" <<'PY'
import sys
from paper_1808_02638_b200 import build
name, defs = sys.argv[1], tuple(sys.argv[2:])
print(build.build(force=True, defs=defs, out=f"build/variants/libclaw_{name}.so"))
PY
