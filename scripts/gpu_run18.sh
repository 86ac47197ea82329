for th in 64 128 256 512; do
echo "threads $th"
FLYKV_THREADS=$th VARIANTS="1:1,1:2,1:3,1:4,1:6,1:8,0:1,0:2,0:3,0:4" python scripts/variants.py c2 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' '.join(f'{k}={v[\"GBps\"]:.0f}' if isinstance(v, dict) else f'{k}={v}' for k,v in d.items() if k.startswith('impl')))"
done
