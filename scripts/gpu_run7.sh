mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny or mixed_plan or variants and 8-4-8 or waves" > gpurun_out/sanitizer_memcheck.log 2>&1; echo memcheck rc=$?
tail -4 gpurun_out/sanitizer_memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny or mixed_plan" > gpurun_out/sanitizer_racecheck.log 2>&1; echo racecheck rc=$?
tail -4 gpurun_out/sanitizer_racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny or mixed_plan" > gpurun_out/sanitizer_synccheck.log 2>&1; echo synccheck rc=$?
tail -4 gpurun_out/sanitizer_synccheck.log
