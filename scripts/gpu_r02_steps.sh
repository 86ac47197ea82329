#!/bin/bash
# Per-step reshard kernel times (directions alternate) on c3i and c4, twice each.
cd "$GRAFT_REPO_ROOT"
for cfg in "c3i --requests 64" c4 "c3i --requests 64" c4; do
timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:30], d['reshard_kernel_ms'], d['reshard_kernel_ms_steps'], d['clocks']['reasons'])"
done
