#!/bin/bash
# Does the nvidia-smi clock sampler cause the timed region's outlier steps?
# Same c4 bench with and without it, alternated; then the default line once.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/r02_clk_ab.jsonl
for k in 1 2 3; do
for ms in 200 0; do
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --clock-ms $ms 2>/dev/null | python -c "
import sys,json; d=json.loads(sys.stdin.read())
print(json.dumps({'clock_ms':$ms,'kern_mean':d['reshard_kernel_ms'],'p50_p90':d['reshard_kernel_ms_p50_p90'],'frac':d['roofline']['frac'],'e2e_p50':d['e2e']['switch_latency_ms_p50'],'e2e_p99':d['e2e']['switch_latency_ms_p99'],'clocks':d['clocks'],'tail':d['e2e']['latency_breakdown']}))" >> gpurun_out/r02_clk_ab.jsonl
done; done
cat gpurun_out/r02_clk_ab.jsonl
