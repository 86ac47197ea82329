# R20: the long-context promotion (config 5, longest request last) in block-aligned pieces with 41% smaller pools
# than one shot, where request-granular waves fail; plus regressions of the default and waves paths.
mkdir -p gpurun_out
: > gpurun_out/pieces.jsonl
timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.2 --long-last --lifo --pieces --steps 6 --warmup 3 --no-cpu-baseline >> gpurun_out/pieces.jsonl 2> gpurun_out/pieces_c5.err; echo c5pieces rc=$?; tail -2 gpurun_out/pieces_c5.err
timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.2 --long-last --lifo --waves --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2> gpurun_out/pieces_c5w.err; echo c5waves-tight rc=$? "(expected to fail: OUT_OF_BLOCKS)"; tail -1 gpurun_out/pieces_c5w.err
timeout 900 python bench.py --config c5 --frag 1.0 --pool-slack 0.55 --waves --steps 6 --warmup 3 --no-cpu-baseline >> gpurun_out/pieces.jsonl 2> gpurun_out/pieces_c5w2.err; echo c5waves rc=$?
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline >> gpurun_out/pieces.jsonl 2> gpurun_out/pieces_c2.err; echo c2 rc=$?
