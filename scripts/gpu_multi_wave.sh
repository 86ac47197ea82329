# kv_switch_multi (every wave in one C call, one sync): parity of the waves / pieces paths, then config 5 in
# waves and in pieces end to end (compare profiles/r01_b_c5waves.json, r01_b_c5pieces.json: one kv_switch per wave).
mkdir -p gpurun_out; : > gpurun_out/mw_ab.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "waves or pieces or kv_switch" > gpurun_out/pytest_mw.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_mw.log
timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.55 --waves --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_c5waves.json 2> gpurun_out/b_c5waves.err; echo c5waves rc=$?; tail -2 gpurun_out/b_c5waves.err
timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.2 --long-last --lifo --pieces --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/b_c5pieces.json 2> gpurun_out/b_c5pieces.err; echo c5pieces rc=$?; tail -2 gpurun_out/b_c5pieces.err
for rep in 1 2; do for m in 1 0; do
FLYKV_MULTI_WAVE=$m timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.55 --waves --steps 10 --warmup 3 --no-cpu-baseline --no-cpu-parallel 2>/dev/null | sed "s/^/M$m /" >> gpurun_out/mw_ab.jsonl
FLYKV_MULTI_WAVE=$m timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.2 --long-last --lifo --pieces --steps 6 --warmup 3 --no-cpu-baseline --no-cpu-parallel 2>/dev/null | sed "s/^/M$m /" >> gpurun_out/mw_ab.jsonl
done; done
