#!/bin/bash
# Atoms in flight per warp (FLYKV_U) x warps per SM on c4, at about 48 KiB in flight per SM and around it.
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
for cfg in "2 192 1" "3 128 1" "3 96 1" "3 64 2" "4 96 1" "4 64 1" "4 128 1"; do
set -- $cfg
FLYKV_U=$1 FLYKV_THREADS=$2 FLYKV_CTAS=$3 timeout 600 python bench.py --steps 16 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print('U $1 threads $2 ctas $3', d['reshard_kernel_ms'], d['reshard_kernel_ms_p50_p90'], d['roofline']['frac'])"
done; done
