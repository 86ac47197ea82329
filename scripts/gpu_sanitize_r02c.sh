#!/bin/bash
# racecheck / synccheck / memcheck of the final replica defaults: TMA <4,1> (8 replicas), <3,1> (4), LDG replica-major (2).
cd "$GRAFT_REPO_ROOT"
K="grid_ragged and (1-1-8 or 2-1-8 or 4-1-8 or 2-2-8 or 1-2-8)"
for tool in racecheck synccheck memcheck; do
timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "$K" > gpurun_out/r02_sanitizer_final_$tool.log 2>&1; echo $tool rc=$?
tail -2 gpurun_out/r02_sanitizer_final_$tool.log
done
