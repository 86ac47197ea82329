# One B200: every BASELINE config shape with virtual ranks (request prefixes
# where the full set does not fit one GPU's HBM).
mkdir -p gpurun_out
: > gpurun_out/sweep.jsonl
run() { timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" >> gpurun_out/sweep.jsonl 2>> gpurun_out/sweep.err; echo "$@ rc=$?"; }
run --config tiny
run --config c2
run --config c4
run --config c4fan
run --config c4gqa4
run --config c4gqa2
run --config c4gqa1
run --config c3i --requests 64
run --config c3ii --requests 64
run --config c5 --requests 33
run --config single
