#!/bin/bash
# Build search-kernel variants (CTA size / min resident CTAs) into tools/variants/<name>/libbmc_b200.so
# usage: tools/build_variants.sh name:THREADS:MINB [...]
cd "$(dirname "$0")/../paper_2508_05990_b200/csrc"
for spec in "$@"; do
  IFS=: read name th mb <<< "$spec"
  out=/root/repo/tools/variants/$name; mkdir -p $out /tmp/vobj_$name
  ( for f in bmc_api bmc_fme bmc_fme_k_u8c4 bmc_fme_k_u8c2 bmc_fme_k_u16 bmc_fme_small bmc_ops; do
      nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
        -DBMC_STAGE_THREADS=$th -DBMC_STAGE_MINB=$mb -I ../../include -c $f.cu -o /tmp/vobj_$name/$f.o &
    done; wait
    nvcc -gencode arch=compute_100a,code=sm_100a --shared -o $out/libbmc_b200.so /tmp/vobj_$name/*.o ) &
done
wait
ls -la /root/repo/tools/variants/*/
