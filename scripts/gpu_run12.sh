timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; tail -2 gpurun_out/bench.err
bash scripts/sweep.sh
FLYKV_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --steps 10 --warmup 3 > gpurun_out/bench_n2_samedev.json 2> gpurun_out/bench_n2_samedev.err; echo benchn2 rc=$?
tail -2 gpurun_out/bench_n2_samedev.err
