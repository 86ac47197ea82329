#!/bin/bash
# For a multi-GPU (NVSwitch) box -- not runnable on the one-GPU gpurun boxes:
# the strong-scaling series of the headline switch, the weak-scaling series, the NCCL all-to-all
# comparator, the NVLS multicast path for GQA replicas, the NVLS parity test,
# and NVLink tx/rx bytes of one rank's push kernel (ncu metric names checked
# offline with `ncu --query-metrics --chip gb100`).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
n=$(nvidia-smi -L | wc -l)
: > gpurun_out/scale.jsonl
for g in 1 2 4 8; do
  [ "$g" -le "$n" ] || continue
  timeout 900 python bench.py --gpus $g --steps 20 --warmup 5 >> gpurun_out/scale.jsonl 2> gpurun_out/scale_n$g.err; echo "c4 N=$g rc=$?"
  grep -c "NCCL INFO.*nranks $g" gpurun_out/scale_n$g.err
done
for g in 1 2 4 8; do   # weak-scaling series: per-GPU bytes fixed
  [ "$g" -le "$n" ] || continue
  timeout 900 python bench.py --gpus $g --config weak --steps 20 --warmup 5 >> gpurun_out/scale.jsonl 2>/dev/null; echo "weak N=$g rc=$?"
done
for g in 2 8; do
  [ "$g" -le "$n" ] || continue
  timeout 900 python bench.py --gpus $g --config c4 --a2a --steps 10 --warmup 3 --no-e2e >> gpurun_out/scale.jsonl 2>/dev/null; echo "a2a N=$g rc=$?"
  timeout 900 python bench.py --gpus $g --config c4gqa1 --steps 10 --warmup 3 >> gpurun_out/scale.jsonl 2>/dev/null; echo "gqa1 N=$g rc=$?"
  timeout 900 python bench.py --gpus $g --config c4gqa1 --nvls --steps 10 --warmup 3 >> gpurun_out/scale.jsonl 2>/dev/null; echo "gqa1 nvls N=$g rc=$?"
done
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -rs -k nvls > gpurun_out/pytest_nvls_mgpu.log 2>&1; echo "nvls parity rc=$?"
# NVLink bytes of rank 0's push kernel, 2 ranks (profile rank 0 only)
if [ "$n" -ge 2 ]; then
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29555 \
    --no-python bash -c 'if [ "$RANK" = 0 ]; then exec ncu --metrics gpu__time_duration.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:flykv_reshard -s 4 -c 2 --csv --log-file gpurun_out/ncu_nvlink_rank0.csv python bench.py --gpus 2 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline; else exec python bench.py --gpus 2 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline; fi' > gpurun_out/ncu_nvlink.log 2>&1
  echo "ncu nvlink rc=$?"
fi
