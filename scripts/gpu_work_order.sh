# Work order (kv_cache_set_work_order): parity of both orders, and the
# single-GPU cost of the mixed order (virtual ranks: no links, so the order
# should not matter there) on the c2 / c4 bench workloads.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
: > gpurun_out/work_order.jsonl
for cfg in c4gqa1 c4gqa4 c2 c4; do
  for wo in 1 0; do
    timeout 600 python bench.py --config $cfg --work-order $wo --steps 20 --warmup 3 --no-cpu-baseline --no-cpu-parallel >> gpurun_out/work_order.jsonl 2>> gpurun_out/work_order.err; echo $cfg $wo rc=$?
  done
done
