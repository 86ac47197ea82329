echo "host: $(nproc) cores, $(free -g | awk "/Mem:/{print \$2}") GB RAM"
# Full measurement pass: tests, smoke, default bench, 1-GPU sweep, ncu launch list + full capture.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; cat gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_ref.json 2>&1; echo ref rc=$?
bash scripts/sweep.sh
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --profile-steps 4 --no-fill > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flykv_reshard -s 2 -c 1 -o gpurun_out/prof_reshard_c2_full python bench.py --profile-steps 3 --no-fill > gpurun_out/ncu_full_c2.log 2>&1; echo ncu2 rc=$?
for n in 2 4 8; do
FLYKV_SAME_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2951$n bench.py --steps 10 --warmup 3 > gpurun_out/bench_n${n}_samedev.json 2> gpurun_out/bench_n${n}_samedev.err; echo benchn$n rc=$?
done
