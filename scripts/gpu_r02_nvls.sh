#!/bin/bash
# NVLS path on one GPU: emulated team addressing, capability report, VMM pool
# exchange through POSIX handles (processes sharing cuda:0), bench --nvls report.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "multicast or nvls or strict or failed_wave" -rs > gpurun_out/pytest_nvls.log 2>&1; echo pytest1 rc=$?; tail -5 gpurun_out/pytest_nvls.log
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q -x -rs > gpurun_out/pytest_mp.log 2>&1; echo pytest2 rc=$?; tail -5 gpurun_out/pytest_mp.log
FLYKV_SAME_DEVICE=1 timeout 600 python bench.py --gpus 2 --config c4gqa1 --steps 3 --warmup 3 --nvls --no-e2e > gpurun_out/r02_nvls_samedev.json 2> gpurun_out/r02_nvls_samedev.err; echo bench rc=$?; python -c "import json;d=json.load(open('gpurun_out/r02_nvls_samedev.json'));print(d['nvls'], d['config']['workload'], d['value'])"; tail -3 gpurun_out/r02_nvls_samedev.err
