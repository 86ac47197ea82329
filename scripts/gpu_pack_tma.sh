# kv_pack through the TMA bulk ring (kv_set_reshard_impl(2)): parity of every variant as reshard and as pack, and the pack cost next to the LDG pack.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "variants or pack_all_to_all" > gpurun_out/pytest_pack_tma.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_pack_tma.log
: > gpurun_out/pack_tma.jsonl
for cfg in c2 c4 c4gqa4; do
VARIANTS="0:0,2:0" timeout 600 python scripts/variants.py $cfg 2>/dev/null | tail -1 >> gpurun_out/pack_tma.jsonl; echo $cfg rc=$?
done
