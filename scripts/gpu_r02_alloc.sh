#!/bin/bash
# After the allocator cursor / word-wise bit sets and the recycled table buffers: parity, then e2e.
cd "$GRAFT_REPO_ROOT"
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_alloc.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_alloc.log
for c in c4 c4gqa1 c5; do
timeout 600 python bench.py --config $c --steps 16 --warmup 4 --no-cpu-baseline $( [ $c = c5 ] && echo --frag 1.0 ) 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read()); e=d['e2e']
print('$c', d['reshard_kernel_ms_forward_reverse'], e['switch_latency_ms_p50'], e['switch_latency_ms_p50_forward_reverse'], e['switch_latency_ms_p99'], e['host_plan_ms_p50'], e['latency_breakdown']['median_step'])"
done
