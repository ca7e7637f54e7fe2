#!/bin/bash
# Builds liblbk variants (tile / cap / min-blocks) into build/variants/ for A/B timing.
set -e
cd "$(dirname "$0")/../paper_2011_08879_b200/csrc"
mkdir -p ../../build/variants
for v in "$@"; do
  IFS=, read T C M <<< "$v"
  out=../../build/variants/liblbk_${T}_${C}_${M}.so
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC,-O3 \
    --expt-relaxed-constexpr -I../../include -DLBK_WTILE=$T -DLBK_WCAP=$C -DLBK_MINB=$M \
    -shared -o $out *.cu -lnccl &
done
wait
