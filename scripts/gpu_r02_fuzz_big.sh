#!/bin/bash
# Large randomised campaign on fresh seeds: single-process switches (all launch paths), memory-bounded
# waves / pieces, multi-process switches (ranks sharing the GPU, host barrier).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
FLYKV_FUZZ_CASES=2500 FLYKV_FUZZ_SEED0=200000 FLYKV_FUZZ_WAVE_CASES=400 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/r02_fuzz_big.log 2>&1; echo fuzz rc=$?
tail -3 gpurun_out/r02_fuzz_big.log
FLYKV_MP_FUZZ_CASES=40 timeout 1800 python -m pytest tests/test_gpu_multiproc.py -m gpu -q -x -k rand > gpurun_out/r02_fuzz_mp_big.log 2>&1; echo mp rc=$?
tail -3 gpurun_out/r02_fuzz_mp_big.log
