#!/bin/bash
# usage: tools/sweep_env.sh "c2 c5" "ENV1=a ENV2=b" "ENV1=c" ...   (time_me per config per env setting)
cd "$(dirname "$0")/.."
cfgs=$1; shift
for c in $cfgs; do for e in "$@"; do
  env $e VARIANT="$e" timeout 200 python tools/time_me.py $c 8 2>&1 | tail -1 | cut -c1-120
done; done
