for cfg in c4gqa1 c4gqa4; do for combo in "192 2" "128 3" "128 4" "96 4" "160 2" "224 2"; do
set -- $combo
FLYKV_THREADS=$1 VARIANTS=0:$2 python scripts/variants.py $cfg 2>/dev/null | head -1 > gpurun_out/v.json
python - "$cfg" "$1" "$2" <<'PY'
import json, sys
d = json.load(open("gpurun_out/v.json"))
print(sys.argv[1], "thr", sys.argv[2], "ctas", sys.argv[3], " ".join(f"{k}={v['GBps']:.0f}" for k, v in d.items() if k.startswith("impl")))
PY
done; done
