#!/bin/bash
for v in 0 1; do
  LBK_L2_PERSIST=$v python bench.py --no-cg --no-cpu --no-cfg3 --steps 30 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); f=d['formats']
print('persist=$v', d['value'], {k: (f[k]['us'], f[k]['frac']) for k in f if k.startswith('cfg')})"
  LBK_L2_PERSIST=$v python scripts/prof_cg.py 300
done
