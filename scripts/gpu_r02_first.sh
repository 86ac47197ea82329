#!/bin/bash
# Round 2 first call: device barrier + virtual-rank multiprocess parity,
# the default (c4 headline) bench line, and the self-launched N-rank bench in
# same-device test mode.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q > gpurun_out/r02_multiproc.log 2>&1; echo "multiproc rc=$?"
tail -3 gpurun_out/r02_multiproc.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_c4.json 2> gpurun_out/r02_bench_c4.err; echo "bench rc=$?"
cat gpurun_out/r02_bench_c4.json; tail -5 gpurun_out/r02_bench_c4.err
FLYKV_SAME_DEVICE=1 timeout 600 python bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02_bench_n4_samedev.json 2> gpurun_out/r02_bench_n4_samedev.err; echo "n4 rc=$?"
cat gpurun_out/r02_bench_n4_samedev.json; tail -5 gpurun_out/r02_bench_n4_samedev.err
FLYKV_SAME_DEVICE=1 timeout 600 python bench.py --gpus 2 --steps 5 --warmup 3 --no-fill > gpurun_out/r02_bench_n2_samedev.json 2> gpurun_out/r02_bench_n2_samedev.err; echo "n2 rc=$?"
cat gpurun_out/r02_bench_n2_samedev.json; tail -5 gpurun_out/r02_bench_n2_samedev.err
