#!/bin/bash
# After the GQA default change: parity of every replication path, then the bench lines.
cd "$GRAFT_REPO_ROOT"
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_consumer.py tests/test_gpu_soak.py -q -x > gpurun_out/pytest_gqa_final.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_gqa_final.log
: > gpurun_out/r02_gqa_bench2.jsonl
for cfg in c4gqa1 c4gqa2 c4gqa4; do
timeout 600 python bench.py --config $cfg --steps 16 --warmup 4 --no-cpu-baseline >> gpurun_out/r02_gqa_bench2.jsonl 2>/dev/null; echo $cfg rc=$?
done
FLYKV_REP_TMA=0 FLYKV_REP_FLAGS=1 FLYKV_THREADS=192 timeout 600 python bench.py --config c4gqa2 --steps 16 --warmup 4 --no-cpu-baseline >> gpurun_out/r02_gqa_bench2.jsonl 2>/dev/null; echo ab2 rc=$?
FLYKV_REP_FLAGS=1 FLYKV_THREADS=192 timeout 600 python bench.py --config c4gqa4 --steps 16 --warmup 4 --no-cpu-baseline >> gpurun_out/r02_gqa_bench2.jsonl 2>/dev/null; echo ab4 rc=$?
python - <<'PY'
import json
for line in open("gpurun_out/r02_gqa_bench2.jsonl"):
    d = json.loads(line); c = d["config"]
    print(c["workload"][:40], d["reshard_kernel_ms"], d["roofline"]["frac"], d["e2e"]["switch_latency_ms_p50"], d["roofline"]["kernel"][:30])
PY
