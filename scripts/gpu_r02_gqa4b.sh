#!/bin/bash
# H_kv=4 -> TP8 forward: around the 8-warp serial-replica optimum, interleaved twice.
cd "$GRAFT_REPO_ROOT"
for rep in 1 2; do
for cfg in "1 192 1" "0 256 1" "0 128 2" "0 224 1" "2 224 1" "0 160 2" "2 256 1" "0 96 3"; do
set -- $cfg
FLYKV_REP_FLAGS=$1 FLYKV_THREADS=$2 FLYKV_CTAS=$3 VARIANTS="0:0" timeout 600 python scripts/variants.py c4gqa4 2>/dev/null | head -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); v=d['impl0_ctas0']; print('rep_flags $1 threads $2 ctas $3: %.3f ms %.0f GB/s' % (v['ms'], v['GBps']))"
done; done
