#!/bin/bash
# Dev tool: build libmpgabor with extra nvcc flags into paper_2202_12380_b200/libmpgabor_<tag>.so
# for A/B timing (MPGABOR_LIB=<path> python tools/...).  usage: tools/build_variant.sh <tag> -DFOO ...
set -e
cd "$(dirname "$0")/.."
tag=$1; shift
python - "$tag" "$@" <<'PY'
import sys
from paper_2202_12380_b200.build import build_library, _HERE
import os
tag, flags = sys.argv[1], sys.argv[2:]
print("built", build_library(extra=flags, out=os.path.join(_HERE, f"libmpgabor_{tag}.so")))
PY
