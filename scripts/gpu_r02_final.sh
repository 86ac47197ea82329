#!/bin/bash
# Round-2 final pass: GPU suite, smoke, default bench (c4 headline), reference arm, decode line,
# ncu launch list of the default bench.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
timeout 900 python bench.py --decode --steps 20 --warmup 5 > gpurun_out/r02_decode.json 2> gpurun_out/r02_decode.err; echo decode rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c4_final.csv python bench.py --profile-steps 4 --no-fill > gpurun_out/ncu_launch.log 2>&1; echo ncu rc=$?
