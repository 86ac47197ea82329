#!/bin/bash
# Multi-process tests on one GPU with the host barrier; the device barrier's
# cooperative-launch emulation; the C demo; same-device bench N=2/4.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_c_example.py -m gpu -q -x -rs > gpurun_out/pytest_mp.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_mp.log
for n in 2 4; do
FLYKV_SAME_DEVICE=1 timeout 600 python bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r02_bench_n${n}_samedev_hostbar.json 2> gpurun_out/r02_bench_n${n}_samedev_hostbar.err; echo benchn$n rc=$?
tail -c 600 gpurun_out/r02_bench_n${n}_samedev_hostbar.json
done
