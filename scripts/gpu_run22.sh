run() { FLYKV_BENCH_DEBUG=1 timeout 900 python bench.py --no-cpu-baseline --steps 20 "$@" > gpurun_out/bench.json 2>gpurun_out/bench.err; echo "args: $@"; grep "e2e per-step" gpurun_out/bench.err | cut -c1-200; }
run
run --clock-ms 0
run --no-fill
run --clock-ms 0 --no-fill
