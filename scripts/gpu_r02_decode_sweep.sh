#!/bin/bash
# N3 decode: consumer parity, then a launch-shape sweep (warps/CTA, CTAs/SM, split tokens; rebuilds the
# library per shape).  SWEEP="w,c,s w,c,s ..."
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_consumer.py -m gpu -q -x > gpurun_out/pytest_consumer.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_consumer.log
: > gpurun_out/r02_decode_sweep.txt
for cfg in ${SWEEP:-4,2,256 4,2,512 4,2,128 2,4,256 8,1,512}; do
  IFS=, read w c sp pr kp <<< "$cfg"
  FLYKV_NVCC_EXTRA="-DFLYKV_DEC_WARPS=$w -DFLYKV_DEC_CTAS=$c -DFLYKV_DEC_SPLIT=$sp -DFLYKV_DEC_PAIR=${pr:-0} -DFLYKV_DEC_KPREF=${kp:-1}" python -c "from paper_2602_22593_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || echo build failed $cfg
  r=$(timeout 600 python bench.py --decode --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['roofline']['frac'], d['dp_layout']['ms_per_step'], d['dp_layout']['frac'])")
  echo "warps $w ctas/SM $c split $sp pair ${pr:-0} kpref ${kp:-1}: tp ms frac / dp ms frac = $r" | tee -a gpurun_out/r02_decode_sweep.txt
done
python -c "from paper_2602_22593_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
