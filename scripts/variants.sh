#!/bin/bash
# Builds liblbk variants for A/B timing: each argument is a list of
# -D defines separated by commas, e.g.  LBK_CSR_CAP=768,LBK_COO_CAP=512
set -e
cd "$(dirname "$0")/../paper_2011_08879_b200/csrc"
mkdir -p ../../_variants
for v in "$@"; do
  defs=""
  for d in ${v//,/ }; do defs="$defs -D$d"; done
  out=../../_variants/liblbk_${v//[=,]/_}.so
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++20 -Xcompiler -fPIC,-O3 \
    --expt-relaxed-constexpr -I../../include $defs -shared -o $out *.cu *.cpp -ldl &
done
wait
ls ../../_variants
