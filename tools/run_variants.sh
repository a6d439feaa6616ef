#!/bin/bash
# Time the ME launch of each config with the in-tree library and every tools/variants/*/libbmc_b200.so.
# usage: tools/run_variants.sh "c2 c5" [reps]
cd "$(dirname "$0")/.."
cfgs=${1:-c2}; reps=${2:-8}
for c in $cfgs; do VARIANT=default timeout 300 python tools/time_me.py $c $reps 2>&1 | tail -1; done
for d in ${VARDIR:-tools/variants}/*/; do
  n=$(basename $d)
  for c in $cfgs; do VARIANT=$n VARIANT_LIB=$PWD/$d/libbmc_b200.so timeout 300 python tools/time_me.py $c $reps 2>&1 | tail -1; done
done
