# Re-measure the full-size long-context promotion (config 5), one-shot and in waves, and the single-request promotion.
mkdir -p gpurun_out
timeout 900 python bench.py --config c5 --frag 1.0 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_c5full.json 2> gpurun_out/b_c5full.err; echo c5full rc=$?; tail -3 gpurun_out/b_c5full.err
timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.55 --waves --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_c5waves.json 2> gpurun_out/b_c5waves.err; echo c5waves rc=$?; tail -3 gpurun_out/b_c5waves.err
timeout 600 python bench.py --config single --steps 40 --warmup 4 --no-cpu-baseline > gpurun_out/b_single.json 2> gpurun_out/b_single.err; echo single rc=$?
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
