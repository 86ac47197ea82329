for cfg in c2 c4; do
for combo in "192 1" "96 2" "64 3" "32 6" "160 1" "224 1" "256 1" "128 1"; do
set -- $combo
r=$(FLYKV_THREADS=$1 VARIANTS="0:$2,0:$2,0:$2" python scripts/variants.py $cfg 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' '.join(f'{v[\"GBps\"]:.0f}' for k,v in d.items() if k.startswith('impl')))")
echo "$cfg thr=$1 ctas=$2 warps/SM=$(( $1 * $2 / 32 )) : $r"
done
done
