for n in 4 8; do
FLYKV_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2952$n bench.py --steps 6 --warmup 3 > gpurun_out/bench_n${n}_samedev.json 2> gpurun_out/bench_n${n}_samedev.err; echo benchn$n rc=$?
tail -2 gpurun_out/bench_n${n}_samedev.err | cut -c1-300
python -c "
import json; d=json.loads(open('gpurun_out/bench_n${n}_samedev.json').read()); c=d['config']
print(d['n_gpus'], c['workload'], d['value'], d['ms_per_step'], d['reshard_kernel_ms'], d['roofline']['bound'], d['roofline']['frac'], d['e2e'])"
done
