# Default bench plus the torchrun path with ranks sharing cuda:0 (gloo barrier), mixed work order.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
for n in 2 8; do
FLYKV_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --steps 6 --warmup 3 --work-order 1 > gpurun_out/bench_n${n}_samedev_mixed.json 2> gpurun_out/bench_n${n}_samedev_mixed.err; echo benchn$n rc=$?
done
