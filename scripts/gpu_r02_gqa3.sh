#!/bin/bash
# After making the lane-parallel TMA ring the default for >= 8 replicas: parity, bench, ncu.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_consumer.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_parity.log
: > gpurun_out/r02_gqa_bench.jsonl
for cfg in c4gqa1 c4gqa4 c4; do
timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/r02_gqa_bench.jsonl 2>/dev/null; echo $cfg rc=$?
done
FLYKV_REP_TMA=0 timeout 600 python bench.py --config c4gqa1 --steps 10 --warmup 3 --no-cpu-baseline >> gpurun_out/r02_gqa_bench.jsonl 2>/dev/null; echo ab rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flykv_reshard -s 2 -c 1 -o gpurun_out/r02_prof_reshard_c4gqa1_tma python bench.py --config c4gqa1 --profile-steps 3 --no-fill > gpurun_out/r02_ncu_gqa1_tma.log 2>&1; echo ncu1 rc=$?
