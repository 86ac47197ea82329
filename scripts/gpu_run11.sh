for cfg in "--config c5 --requests 33" "--config c4"; do
 for ck in 0 50 200; do
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --clock-ms $ck $cfg 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg clock $ck', d['ms_per_step'], d['reshard_kernel_ms'], d['clocks'])"
 done
done
