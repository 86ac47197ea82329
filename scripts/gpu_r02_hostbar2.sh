#!/bin/bash
# The self-launched multi-rank bench test, strict mode through kv_switch_range,
# and sanitizers over the barrier self-test and the host-barrier one-call path.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_bench.py "tests/test_gpu_parity.py::test_strict_replica_mode" -m gpu -q -x -rs > gpurun_out/pytest_hb2.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_hb2.log
for tool in memcheck racecheck synccheck; do
timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python -m pytest -q -m gpu -x \
  "tests/test_gpu_multiproc.py::test_device_barrier_emulated_members" \
  "tests/test_gpu_multiproc.py::test_device_barrier_absent_member_times_out" \
  "tests/test_gpu_multiproc.py::test_device_barrier_prearrived_launch" > gpurun_out/r02_sanitizer_barrier_$tool.txt 2>&1; echo $tool rc=$?
tail -3 gpurun_out/r02_sanitizer_barrier_$tool.txt
done
