for c in c2 c4 c3ii c3i; do for r in "" 1; do
REVERSE=$r VARIANTS=0:0,1:0 python scripts/variants.py $c 2>/dev/null | tail -1 > /tmp/v.json
python - "$c" "$r" <<'PY'
import json, sys
d = json.load(open("/tmp/v.json"))
print(sys.argv[1], "reverse" if sys.argv[2] else "forward", " ".join(f"{k}={v['GBps']:.0f}" for k, v in d.items() if k.startswith("impl")))
PY
done; done
