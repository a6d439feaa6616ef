#!/bin/bash
# ME timing sweep: in-tree lib + each variant, several BMC_MAX_THREADS caps.  usage: tools/sweep_c2.sh "c2 c5" "416 256 224 128"
cd "$(dirname "$0")/.."
cfgs=${1:-c2}; caps=${2:-"416 256 224 160 128"}
for c in $cfgs; do for mt in $caps; do
  BMC_MAX_THREADS=$mt VARIANT="default_mt$mt" timeout 200 python tools/time_me.py $c 8 2>&1 | tail -1
  for d in tools/variants/*/; do n=$(basename $d)
    VARIANT_LIB=$PWD/$d/libbmc_b200.so BMC_MAX_THREADS=$mt VARIANT="${n}_mt$mt" timeout 200 python tools/time_me.py $c 8 2>&1 | tail -1
  done
done; done
