#!/bin/bash
# Build search-kernel CTA-shape variants into tools/variants/<name>/libbmc_b200.so
set -e
cd "$(dirname "$0")/.."
for v in "256 2" "128 4" "256 3" "128 3" "384 1" "192 2"; do
  set -- $v
  d=tools/variants/t$1_b$2; mkdir -p $d
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared -Xcompiler -fPIC \
    -DBMC_SEARCH_THREADS=$1 -DBMC_SEARCH_MINB=$2 -I include -o $d/libbmc_b200.so \
    paper_2508_05990_b200/csrc/bmc_api.cu paper_2508_05990_b200/csrc/bmc_fme.cu paper_2508_05990_b200/csrc/bmc_ops.cu &
done
wait
