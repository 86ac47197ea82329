#!/bin/bash
# Launch-shape re-check of the LDG/STG reshard on the headline c4 (threads x CTAs/SM), interleaved twice.
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
for shape in "192 1" "160 1" "224 1" "128 2" "96 2" "160 2" "256 1"; do
set -- $shape
FLYKV_THREADS=$1 FLYKV_CTAS=$2 timeout 600 python bench.py --steps 16 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('threads $1 ctas $2', d['reshard_kernel_ms'], d['reshard_kernel_ms_p50_p90'], d['roofline']['frac'])"
done; done
