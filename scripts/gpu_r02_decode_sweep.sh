#!/bin/bash
# N3 decode: consumer parity of the default build, then variants given as SWEEP="K=V,K=V ..." (each K
# becomes -DFLYKV_DEC_K=V; the library is rebuilt per variant), each timed with bench.py --decode.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
: > gpurun_out/r02_decode_sweep.txt
for cfg in ${SWEEP:-STAGE=0}; do
  flags=$(echo "$cfg" | tr ',' '\n' | sed 's/^/-DFLYKV_DEC_/' | tr '\n' ' ')
  FLYKV_NVCC_EXTRA="$flags" python -c "from paper_2602_22593_b200 import _build; _build.build(force=True)" > /dev/null 2>&1 || echo build failed $cfg
  t=$(timeout 600 python -m pytest tests/test_gpu_consumer.py -m gpu -q -x 2>&1 | tail -1)
  r=$(timeout 600 python bench.py --decode --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['roofline']['frac'], d['dp_layout']['ms_per_step'], d['dp_layout']['frac'])")
  echo "$cfg: tp ms frac / dp ms frac = $r   [consumer: $t]" | tee -a gpurun_out/r02_decode_sweep.txt
done
python -c "from paper_2602_22593_b200 import _build; _build.build(force=True)" > /dev/null 2>&1
