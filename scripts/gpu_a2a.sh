# pack -> all-to-all -> unpack path: parity (single process, multi-process gloo), then its HBM cost next to the fused kernel.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "pack_all_to_all or full_size" > gpurun_out/pytest_a2a.log 2>&1; echo pytest1 rc=$?; tail -1 gpurun_out/pytest_a2a.log
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x -k a2a > gpurun_out/pytest_a2a_mp.log 2>&1; echo pytest2 rc=$?; tail -1 gpurun_out/pytest_a2a_mp.log
: > gpurun_out/a2a.jsonl
for cfg in c2 c4gqa4 c4gqa1; do
VARIANTS="0:0" timeout 600 python scripts/variants.py $cfg 2>/dev/null | tail -1 >> gpurun_out/a2a.jsonl; echo $cfg rc=$?
done
REVERSE=1 VARIANTS="0:0" timeout 600 python scripts/variants.py c2 2>/dev/null | tail -1 >> gpurun_out/a2a.jsonl; echo c2rev rc=$?
