for r in "" 1; do for th in 128 192 256; do for ct in 1 2; do
FLYKV_THREADS=$th REVERSE=$r VARIANTS=0:$ct python scripts/variants.py c4gqa1 2>/dev/null | head -1 > gpurun_out/v.json
python - "$r" "$th" "$ct" <<'PY'
import json, sys
d = json.load(open("gpurun_out/v.json"))
print("reverse" if sys.argv[1] else "forward", "thr", sys.argv[2], "ctas", sys.argv[3], " ".join(f"{k}={v['GBps']:.0f}" for k, v in d.items() if k.startswith("impl")))
PY
done; done; done
