timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b1.json 2> gpurun_out/b1.err; echo rc=$?; tail -2 gpurun_out/b1.err
for cfg in "--config c5 --frag 1.0" "--config c5 --frag 1.0 --rank-ids suggest" "--config c3ii --requests 64" "--config c3ii --requests 64 --rank-ids suggest" "--config c4"; do
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --no-e2e $cfg > gpurun_out/bx.json 2> gpurun_out/bx.err; echo "$cfg rc=$?"; tail -1 gpurun_out/bx.err
python -c "
import json; d=json.loads(open('gpurun_out/bx.json').read()); print(d['config']['workload'], d['reshard_kernel_ms'], d['roofline']['frac'], d['modeled_nvlink'])"
done
FLYKV_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --steps 5 --warmup 3 --rank-ids suggest > gpurun_out/bn4.json 2> gpurun_out/bn4.err; echo n4 rc=$?; tail -2 gpurun_out/bn4.err | cut -c1-200
