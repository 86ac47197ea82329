for cfg in c2 c4; do
for th in 32 64 96 128; do
echo "$cfg threads $th"
FLYKV_THREADS=$th VARIANTS="0:2,0:3,0:4,0:5,0:6,0:8,1:4,1:6,1:8" python scripts/variants.py $cfg 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' '.join(f'{k}={v[\"GBps\"]:.0f}' if isinstance(v, dict) else f'{k}=ERR' for k,v in d.items() if k.startswith('impl')))"
done
done
