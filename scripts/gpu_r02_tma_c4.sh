#!/bin/bash
# TMA ring shapes at many occupancies on the copy-like headline (1 replica), against the LDG default.
cd "$GRAFT_REPO_ROOT"
for shape in 16 10 13 11 12 0; do
FLYKV_TMA_SHAPE=$shape VARIANTS="0:0,2:2,2:4,2:6,2:8,2:10,2:12,2:16" timeout 600 python scripts/variants.py c4 2>/dev/null | head -8 | tail -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('c4 tma shape $shape', {k: (round(v['ms'],3) if isinstance(v, dict) else v[:20]) for k, v in d.items() if k.startswith('impl')})"
done
