#!/bin/bash
# H_kv=4 -> TP8 (2 replicas) forward plan: replica store strategy x launch shape x atoms in flight.
cd "$GRAFT_REPO_ROOT"
: > gpurun_out/r02_gqa4_sweep.txt
for rf in 0 1 2 3; do
for cfg in "2 192 1" "2 96 2" "2 256 1" "3 128 1" "4 128 1"; do
set -- $cfg
FLYKV_REP_FLAGS=$rf FLYKV_U=$1 FLYKV_THREADS=$2 FLYKV_CTAS=$3 VARIANTS="0:0" timeout 600 python scripts/variants.py c4gqa4 2>/dev/null | head -1 | python -c "
import sys,json; d=json.loads(sys.stdin.read()); v=d['impl0_ctas0']; print('rep_flags $rf U $1 threads $2 ctas $3: %.3f ms %.0f GB/s' % (v['ms'], v['GBps']))" | tee -a gpurun_out/r02_gqa4_sweep.txt
done; done
