# kv_switch / kv_switch_back (one-call switch): parity, then e2e latency on a few configs.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "kv_switch" > gpurun_out/pytest_switch.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_switch.log
: > gpurun_out/switch.jsonl
for cfg in tiny c2 single c4; do
timeout 600 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline >> gpurun_out/switch.jsonl 2>gpurun_out/switch_$cfg.err; echo $cfg rc=$?
done
timeout 600 python bench.py --config c5 --frag 1.0 --pool-slack 0.55 --waves --steps 6 --warmup 3 --no-cpu-baseline >> gpurun_out/switch.jsonl 2>gpurun_out/switch_c5w.err; echo c5waves rc=$?
