#!/bin/bash
# A/B over _variants/*.so: cfg1/cfg2 SpMV, power-law, CG timing.
for v in _variants/*.so; do
  echo "== $v"
  LBK_LIB=$PWD/$v python scripts/ab_spmv.py 2>&1 | grep -v "^$"
  LBK_LIB=$PWD/$v python scripts/ab_powerlaw.py 10000 2>&1 | grep csr
  LBK_LIB=$PWD/$v python scripts/prof_cg.py 300 2>&1 | tail -1
done
