#!/bin/bash
# H_kv=2 -> TP8 (4 replicas) and H_kv=4 (2 replicas) forward plans: replica strategy x launch shape.
cd "$GRAFT_REPO_ROOT"
for cfgname in c4gqa2 c4gqa4; do
for cfg in "1 192 1" "2 224 1" "0 224 1" "2 256 1" "0 256 1" "2 192 1"; do
set -- $cfg
FLYKV_REP_FLAGS=$1 FLYKV_THREADS=$2 FLYKV_CTAS=$3 VARIANTS="0:0" timeout 600 python scripts/variants.py $cfgname 2>/dev/null | head -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); v=d['impl0_ctas0']; print('$cfgname rep_flags $1 threads $2 ctas $3: %.3f ms %.0f GB/s' % (v['ms'], v['GBps']))"
done; done
