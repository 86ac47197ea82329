#!/bin/bash
# memcheck over the whole small-size parity suite (every kernel and path except the full-size and
# million-token cases) and the consumer / soak tests, on the final round-2 build.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 3000 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_consumer.py -q -x -k "not full_size and not million and not weight_switches and not many_small" > gpurun_out/r02_sanitizer_memcheck_all.log 2>&1; echo memcheck rc=$?
tail -3 gpurun_out/r02_sanitizer_memcheck_all.log
FLYKV_SOAK_ITERS=300 timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_soak.py -q -x > gpurun_out/r02_sanitizer_memcheck_soak.log 2>&1; echo memcheck_soak rc=$?
tail -3 gpurun_out/r02_sanitizer_memcheck_soak.log
