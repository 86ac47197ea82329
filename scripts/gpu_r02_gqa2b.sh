#!/bin/bash
# 4 replicas (H_kv=2 -> TP8): the lane-parallel TMA ring at low occupancy against the best LDG/STG shape.
cd "$GRAFT_REPO_ROOT"
for shape in 0 10 13 3 4; do
FLYKV_TMA_SHAPE=$shape VARIANTS="2:1,2:2,2:3" timeout 600 python scripts/variants.py c4gqa2 2>/dev/null | head -3 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('c4gqa2 tma shape $shape', {k: round(v['ms'],3) for k, v in d.items() if k.startswith('impl')})"
done
FLYKV_REP_FLAGS=2 FLYKV_THREADS=256 FLYKV_CTAS=1 VARIANTS="0:0" timeout 600 python scripts/variants.py c4gqa2 2>/dev/null | head -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('c4gqa2 ldg rep_flags 2 256x1', round(d['impl0_ctas0']['ms'],3))"
