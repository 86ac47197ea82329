set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
FLYKV_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --steps 5 --warmup 3 > gpurun_out/bench_n2_samedev.json 2> gpurun_out/bench_n2_samedev.err; echo benchn2 rc=$?
tail -3 gpurun_out/bench_n2_samedev.err; cat gpurun_out/bench_n2_samedev.json
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo benchc4 rc=$?
tail -3 gpurun_out/bench_c4.err; cat gpurun_out/bench_c4.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flykv_reshard -s 2 -c 1 -o gpurun_out/prof_reshard_c2_full python bench.py --profile-steps 3 --no-fill > gpurun_out/ncu_full_c2.log 2>&1; echo ncu2 rc=$?
tail -3 gpurun_out/ncu_full_c2.log
