#!/bin/bash
# Build measurement variants of the library (-DBMC_EXPERIMENTS: the BMC_* environment knobs are live)
# into tools/variants/<name>/libbmc_b200.so.   usage: tools/build_variants.sh name[:nvcc-define ...] ...
#   e.g. tools/build_variants.sh exp  t320:-DBMC_STAGE_THREADS=320
# Load one from a tool with VARIANT_LIB=tools/variants/<name>/libbmc_b200.so (tools/_variant.py).
cd "$(dirname "$0")/.."
for spec in "$@"; do
  IFS=: read -r name defs <<< "$spec"
  python - "$name" $defs <<'PY' &
import sys
from pathlib import Path
sys.path.insert(0, ".")
from paper_2508_05990_b200 import build
name, defs = sys.argv[1], sys.argv[2:]
out = Path("tools/variants") / name / "libbmc_b200.so"
build.build(force=True, out=out, extra=["-DBMC_EXPERIMENTS", *defs])
print(out)
PY
done
wait
