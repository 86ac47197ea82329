#!/bin/bash
# N3: the tensor-core paged decode kernel -- parity (consumer tests), its bench line, ncu of one TP launch.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_consumer.py -m gpu -q -x > gpurun_out/pytest_consumer.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_consumer.log
timeout 900 python bench.py --decode --steps 20 --warmup 5 > gpurun_out/r02_decode.json 2> gpurun_out/r02_decode.err; echo decode rc=$?
cat gpurun_out/r02_decode.json; tail -3 gpurun_out/r02_decode.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:paged_decode -s 5200 -c 1 \
  -o gpurun_out/r02_prof_decode python bench.py --decode --steps 1 --warmup 1 > gpurun_out/ncu_decode.log 2>&1; echo ncu rc=$?
