#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
./scripts/probe_mc2 > gpurun_out/r02_probe_mc2.txt 2>&1; echo probe rc=$?; cat gpurun_out/r02_probe_mc2.txt
nvidia-smi -q | grep -i -A3 "fabric" | head -20
ls -la /dev/nvidia-caps-imex-channels 2>&1 | head -3
timeout 600 python scripts/n4_pool_capacity.py > gpurun_out/r02_n4.json 2> gpurun_out/r02_n4.err; echo n4 rc=$?; cat gpurun_out/r02_n4.json; tail -5 gpurun_out/r02_n4.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pack or piece or wave or strict" > gpurun_out/pytest_r02b.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_r02b.log
