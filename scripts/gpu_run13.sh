timeout 600 python -m pytest tests/test_c_example.py -q 2>&1 | tail -2
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_c2.json 2> gpurun_out/b_c2.err; echo c2 rc=$?; tail -3 gpurun_out/b_c2.err
timeout 900 python bench.py --config c5 --frag 1.0 --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/b_c5full.json 2> gpurun_out/b_c5full.err; echo c5full rc=$?; tail -3 gpurun_out/b_c5full.err
timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.55 --waves --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/b_c5waves.json 2> gpurun_out/b_c5waves.err; echo c5waves rc=$?; tail -3 gpurun_out/b_c5waves.err
timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.55 --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/b_c5oneshot.err; echo c5oneshot-small rc=$?; tail -1 gpurun_out/b_c5oneshot.err
for f in b_c2 b_c5full b_c5waves; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read()); c=d['config']
print('$f', c['workload'], round(c['payload_bytes_per_step']/1e9,2), 'GB pools', round(c['pool_bytes']/1e9,1), 'GB waves', c['waves_per_switch'], 'step', d['ms_per_step'], 'kern', d['reshard_kernel_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['switch_latency_ms_p50'], d['e2e']['host_plan_ms_p50'])"; done
