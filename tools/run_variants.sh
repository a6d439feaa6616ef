#!/bin/bash
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
for d in tools/variants/*/; do
  n=$(basename $d)
  for ty in 12 11 8 6; do
    VARIANT=$n BMC_TY_MAX=$ty BMC_LIB_PATH=$PWD/$d/libbmc_b200.so python tools/time_me.py c2 8 2>/dev/null
  done
done
