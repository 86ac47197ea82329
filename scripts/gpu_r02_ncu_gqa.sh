#!/bin/bash
# ncu --set full of one forward launch of each GQA variant on the final defaults.
cd "$GRAFT_REPO_ROOT"
for cfg in c4gqa1 c4gqa2 c4gqa4; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flykv_reshard -s 2 -c 1 -o gpurun_out/r02_prof_final_$cfg python bench.py --config $cfg --profile-steps 3 --no-fill > gpurun_out/ncu_final_$cfg.log 2>&1; echo $cfg rc=$?
done
