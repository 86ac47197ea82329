set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
nproc; free -g | head -2
python -c "import torch;print(torch.cuda.get_device_name(0))"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:flykv --csv --log-file gpurun_out/launches.csv python bench.py --profile-steps 3 --no-fill > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flykv_reshard -s 2 -c 1 -o gpurun_out/prof_reshard_c2_8req python bench.py --profile-steps 3 --no-fill --requests 8 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
ls -la gpurun_out
