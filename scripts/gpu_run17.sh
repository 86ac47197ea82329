for pl in fragmented contiguous; do
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --placement $pl > gpurun_out/bp.json 2> gpurun_out/bp.err; echo "$pl rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bp.json').read()); print('$pl', d['reshard_kernel_ms'], d['roofline']['achieved'], d['roofline']['frac'])"
done
