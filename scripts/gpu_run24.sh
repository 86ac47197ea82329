timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pt.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pt.log
for r in "" 1; do
REVERSE=$r VARIANTS=0:0,1:0,2:0 python scripts/variants.py c2 2>/dev/null | tail -1 > gpurun_out/v.json
python - "$r" <<'PY'
import json, sys
d = json.load(open("gpurun_out/v.json"))
print("reverse" if sys.argv[1] else "forward", " ".join(f"{k}={v.get('GBps', v.get('GBps_of_fused_bytes', 0)):.0f}" for k, v in d.items() if isinstance(v, dict)))
PY
done
