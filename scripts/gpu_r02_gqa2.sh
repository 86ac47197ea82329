#!/bin/bash
# TMA ring shapes at low occupancy for the 8-replica (H_kv=1 -> TP8) forward plan, and both directions.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/r02_gqa_tma2.jsonl
for cfg in c4gqa1; do
for shape in 0 10 11 12 13 14 15 16 17 3 4; do
FLYKV_TMA_SHAPE=$shape VARIANTS="0:0,2:1,2:2,2:3,2:4" timeout 600 python scripts/variants.py $cfg 2>/dev/null | head -5 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); d['tma_shape']=$shape; print(json.dumps(d))" >> gpurun_out/r02_gqa_tma2.jsonl; echo $cfg $shape rc=$?
done; done
for shape in 0 10 13; do
REVERSE=1 FLYKV_TMA_SHAPE=$shape VARIANTS="0:0,2:1,2:2,2:3" timeout 600 python scripts/variants.py c4gqa1 2>/dev/null | head -4 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); d['tma_shape']=$shape; d['reverse']=1; print(json.dumps(d))" >> gpurun_out/r02_gqa_tma2.jsonl; echo rev $shape rc=$?
done
