#!/bin/bash
# Round 2 refresh of the long-context promotion (config 5) at full size: one
# shot, memory-bounded waves (24% smaller pools) and block-aligned pieces (41%
# smaller pools), and the single-request promotion, on the round-2 code.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/r02_c5.jsonl
timeout 900 python bench.py --config c5 --frag 1.0 --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/r02_c5.jsonl 2> gpurun_out/r02_c5a.err; echo c5full rc=$?
timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.55 --waves --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/r02_c5.jsonl 2> gpurun_out/r02_c5b.err; echo c5waves rc=$?
timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.2 --long-last --lifo --pieces --steps 6 --warmup 3 --no-cpu-baseline >> gpurun_out/r02_c5.jsonl 2> gpurun_out/r02_c5c.err; echo c5pieces rc=$?
timeout 600 python bench.py --config single --steps 40 --warmup 4 --no-cpu-baseline >> gpurun_out/r02_c5.jsonl 2> gpurun_out/r02_c5d.err; echo single rc=$?
python - <<'PY'
import json
for line in open("gpurun_out/r02_c5.jsonl"):
    if not line.startswith("{"): continue
    d = json.loads(line); c = d["config"]
    print(c["workload"][:40], "waves", c["waves_per_switch"], "pool GB", round(c["pool_bytes"] / 1e9, 1), "kern", d["reshard_kernel_ms"],
          "frac", d["roofline"]["frac"], "e2e p50/p99", d["e2e"]["switch_latency_ms_p50"], d["e2e"]["switch_latency_ms_p99"])
PY
