#!/bin/bash
# Round 2 full measurement pass: GPU tests, smoke, the default bench line (c4
# headline), the reference arm, ncu launch list + one --set full capture of the
# headline reshard launch, self-launched N-rank runs (ranks sharing cuda:0).
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
cat gpurun_out/bench_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c4.csv python bench.py --profile-steps 4 --no-fill > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flykv_reshard -s 2 -c 1 -o gpurun_out/r02_prof_reshard_c4 python bench.py --profile-steps 3 --no-fill > gpurun_out/ncu_full_c4.log 2>&1; echo ncu2 rc=$?
for n in 2 4 8; do
FLYKV_SAME_DEVICE=1 timeout 900 python bench.py --gpus $n --steps 10 --warmup 3 > gpurun_out/r02_bench_n${n}_samedev.json 2> gpurun_out/r02_bench_n${n}_samedev.err; echo benchn$n rc=$?
done
