mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_consumer.py -q -x > gpurun_out/pytest_rep.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pytest_rep.log
: > gpurun_out/gqa_check.jsonl
for cfg in c4gqa1 c4gqa4 c4 c2 c4gqa1 c4gqa4; do
timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'cfg':'$cfg','kernel_ms':d['reshard_kernel_ms'],'TBps':d['roofline']['achieved'],'frac':d['roofline']['frac']}))" >> gpurun_out/gqa_check.jsonl; echo $cfg rc=$?
done
