mkdir -p gpurun_out
: > gpurun_out/a2a_shape.jsonl
for sh in 0 1 2 3; do
FLYKV_UNPACK_SHAPE=$sh VARIANTS="0:0" timeout 600 python scripts/variants.py c2 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); d['unpack_shape']=$sh; print(json.dumps(d))" >> gpurun_out/a2a_shape.jsonl; echo $sh rc=$?
done
