#!/bin/bash
# Finer TMA shape sweep: 2, 4 and 8 replicas.
cd "$GRAFT_REPO_ROOT"
for cfgname in c4gqa4 c4gqa2 c4gqa1; do
for shape in 16 10 13; do
FLYKV_TMA_SHAPE=$shape VARIANTS="2:2,2:4,2:6,2:8,2:10,2:12" timeout 600 python scripts/variants.py $cfgname 2>/dev/null | head -6 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$cfgname tma shape $shape', {k: (round(v['ms'],3) if isinstance(v, dict) else v[:30]) for k, v in d.items() if k.startswith('impl')})"
done; done
