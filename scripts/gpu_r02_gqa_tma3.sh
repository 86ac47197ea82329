#!/bin/bash
# Lane-parallel TMA ring shapes x CTAs/SM for 2 and 4 replicas (forward plans), twice.
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
for cfgname in c4gqa4 c4gqa2; do
for shape in 13 0 16; do
FLYKV_TMA_SHAPE=$shape VARIANTS="2:2,2:3,2:4,2:5,2:6" timeout 600 python scripts/variants.py $cfgname 2>/dev/null | head -5 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('$cfgname tma shape $shape', {k: round(v['ms'],3) for k, v in d.items() if k.startswith('impl') and isinstance(v, dict)})"
done; done; done
