#!/bin/bash
# One ncu --set full capture of a TP-layout decode launch (after the DP warm-ups).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_decode -s 5200 -c 1 \
  -o gpurun_out/r02_prof_decode python bench.py --decode --steps 1 --warmup 1 > gpurun_out/ncu_decode.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ncu_decode.log
