#!/bin/bash
# GQA replication (H_kv=1/4 -> TP8): lane-parallel TMA replica stores vs the
# LDG/STG default, TMA ring shapes; ncu captures of the write-heavy reshard
# launch and of a write-only SM store kernel (the store ceiling).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "variants or (full_size and -2]) or staged" > gpurun_out/pytest_tma.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_tma.log
: > gpurun_out/r02_gqa_tma.jsonl
for cfg in c4gqa1 c4gqa4; do
for shape in 0 1 3 4 5 7 9; do
FLYKV_TMA_SHAPE=$shape VARIANTS="0:0,2:0,2:1,2:2,2:3" timeout 600 python scripts/variants.py $cfg 2>/dev/null | head -5 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); d['tma_shape']=$shape; print(json.dumps(d))" >> gpurun_out/r02_gqa_tma.jsonl; echo $cfg $shape rc=$?
done; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flykv_reshard -s 2 -c 1 -o gpurun_out/r02_prof_reshard_c4gqa1 python bench.py --config c4gqa1 --profile-steps 3 --no-fill > gpurun_out/r02_ncu_gqa1.log 2>&1; echo ncu1 rc=$?
timeout 600 ncu --set full --clock-control none -k regex:w_warp_atom -s 1 -c 1 -o gpurun_out/r02_prof_write_only ./scripts/mbwr > gpurun_out/r02_ncu_wonly.log 2>&1; echo ncu2 rc=$?
timeout 600 ncu --set full --clock-control none -k regex:rep_warp -s 12 -c 1 -o gpurun_out/r02_prof_rep8_micro ./scripts/mbwr > gpurun_out/r02_ncu_rep8.log 2>&1; echo ncu3 rc=$?
