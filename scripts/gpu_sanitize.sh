mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny or mixed_plan or mixed_order or variants and 8-4-8 or waves or rank_ids and 8-4-8 or staged or pack_all_to_all and 8-1-8 or pack_all_to_all and 2-4-8" > gpurun_out/sanitizer_memcheck.log 2>&1; echo memcheck rc=$?
tail -3 gpurun_out/sanitizer_memcheck.log
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny or mixed_plan or mixed_order and per_gpu or variants and 8-4-8" > gpurun_out/sanitizer_racecheck.log 2>&1; echo racecheck rc=$?
tail -3 gpurun_out/sanitizer_racecheck.log
timeout 1200 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "tiny or mixed_plan or variants and 8-4-8 or pack_all_to_all and 8-1-8" > gpurun_out/sanitizer_synccheck.log 2>&1; echo synccheck rc=$?
tail -3 gpurun_out/sanitizer_synccheck.log
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_consumer.py tests/test_c_example.py -q -x > gpurun_out/sanitizer_memcheck2.log 2>&1; echo memcheck2 rc=$?
tail -3 gpurun_out/sanitizer_memcheck2.log
