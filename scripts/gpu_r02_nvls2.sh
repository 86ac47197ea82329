#!/bin/bash
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "multicast or nvls or strict or failed_wave" -rs > gpurun_out/pytest_nvls.log 2>&1; echo pytest1 rc=$?; tail -5 gpurun_out/pytest_nvls.log
