#!/bin/bash
# A/B of the ELL/SELL-P kernels (LBK_SLICED = lane | quad | row) via bench's format sweep
for a in lane quad row; do
  LBK_SLICED=$a python bench.py --no-cg --no-cpu --no-cfg3 --steps 20 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); f=d['formats']
print('$a', {k: (f[k]['us'], f[k]['frac']) for k in f if 'ell' in k or 'sellp' in k})"
done
