for cfg in c4gqa1 c4gqa4; do
for combo in "192 1" "256 1" "256 2" "128 3" "192 2" "256 3"; do
set -- $combo
r=$(FLYKV_THREADS=$1 VARIANTS="0:$2,1:$2" python scripts/variants.py $cfg 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' '.join(f'{k}={v[\"GBps\"]:.0f}' for k,v in d.items() if k.startswith('impl')))")
echo "$cfg thr=$1 ctas=$2 : $r"
done
done
