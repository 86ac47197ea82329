timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x 2>&1 | tail -3
timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.55 --waves --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/b_c5waves.json 2> gpurun_out/b_c5waves.err; echo c5waves rc=$?; tail -3 gpurun_out/b_c5waves.err
python -c "
import json; d=json.loads(open('gpurun_out/b_c5waves.json').read()); c=d['config']
print(c['workload'], round(c['payload_bytes_per_step']/1e9,2), 'GB pools', round(c['pool_bytes']/1e9,1), 'GB waves', c['waves_per_switch'], 'step', d['ms_per_step'], 'kern', d['reshard_kernel_ms'], 'frac', d['roofline']['frac'], 'e2e', d['e2e']['switch_latency_ms_p50'], d['e2e']['host_plan_ms_p50'])"
