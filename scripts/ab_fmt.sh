#!/bin/bash
# A/B of the format sweep (ELL / SELL-P / COO / CSR at cfg2) across the
# in-tree library and every _variants/*.so (LBK_LIB), via bench.py.
for l in default _variants/*.so; do
  if [ $l = default ]; then unset LBK_LIB; else export LBK_LIB=$PWD/$l; fi
  python bench.py --no-cg --no-cpu --no-cfg3 --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); f=d['formats']
print('$(basename $l)', {k.replace('cfg2_',''): (f[k]['us'], f[k]['frac']) for k in f if k.startswith(('cfg1_', 'cfg2_')) and 'conv' not in k})"
done
