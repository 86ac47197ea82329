#!/bin/bash
# Round 2 sanitizer pass over the kernels added or changed this round: the
# lane-parallel TMA replica ring (GQA rep 8 grid cases), the strict-mode
# verify kernel, the device group barrier (2-process case), the NVLS team
# emulation, plus the round-1 set.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
K_NEW="grid_ragged and (1-1-8 or 1-2-8 or 2-1-8) or strict or multicast or failed_wave or tiny or variants and 8-4-8"
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "$K_NEW" > gpurun_out/r02_sanitizer_memcheck.log 2>&1; echo memcheck rc=$?; tail -3 gpurun_out/r02_sanitizer_memcheck.log
timeout 1500 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "grid_ragged and (1-1-8 or 1-2-8) or strict" > gpurun_out/r02_sanitizer_racecheck.log 2>&1; echo racecheck rc=$?; tail -3 gpurun_out/r02_sanitizer_racecheck.log
timeout 1500 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "grid_ragged and (1-1-8 or 1-2-8) or strict" > gpurun_out/r02_sanitizer_synccheck.log 2>&1; echo synccheck rc=$?; tail -3 gpurun_out/r02_sanitizer_synccheck.log
timeout 1500 compute-sanitizer --tool memcheck --target-processes all --print-limit 20 python -m pytest tests/test_gpu_multiproc.py -q -x -k "2-dp_tp-push-1 or 2-dp_tp-vmm" > gpurun_out/r02_sanitizer_memcheck_mp.log 2>&1; echo memcheck_mp rc=$?; tail -3 gpurun_out/r02_sanitizer_memcheck_mp.log
grep -h "ERROR SUMMARY\|RACECHECK SUMMARY\|hazard" gpurun_out/r02_sanitizer_*.log | sort | uniq -c
