mkdir -p gpurun_out
timeout 400 ./scripts/mbwr > gpurun_out/mbwr.txt 2>&1; echo rc=$?
cat > /tmp/ms.py <<'PY'
import torch
x = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
for _ in range(3):
    x.fill_(3)
torch.cuda.synchronize()
PY
timeout 300 ncu --metrics launch__grid_size,launch__block_size,launch__registers_per_thread,dram__bytes_write.sum,gpu__time_duration.sum --csv python /tmp/ms.py > gpurun_out/ncu_fill.csv 2>&1; echo ncu rc=$?
