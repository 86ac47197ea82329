for combo in "256 1" "192 1" "96 2" "64 3" "192 1" "256 1"; do
set -- $combo
python - <<PY
import os, sys, time, json
sys.path.insert(0, ".")
os.environ["FLYKV_THREADS"] = "$1"
import torch, bench, synth
from paper_2602_22593_b200 import flykv as F
from paper_2602_22593_b200.engine import KVSwitchEngine
F.set_reshard_impl(0, $2)
w = synth.WORKLOADS["c2"]()
g = F.geometry(w.L, w.H, w.d, w.B, w.e)
nb, tabs = bench.pools_and_tables(w)
eng = KVSwitchEngine(g, nb, "cuda:0")
for s_, ids in zip(w.src, tabs):
    eng.cache.reserve(s_, ids)
reqs = [(i, T, s_, ids, d) for i, (T, s_, d, ids) in enumerate(zip(w.T, w.src, w.dst, tabs))]
lat = []
for it in range(25):
    t0 = time.perf_counter()
    plan, tables, host = eng.switch(reqs, read_back=True)
    lat.append((time.perf_counter() - t0) * 1e3)
    new = plan.dst_tables()
    reqs = [(rid, T, d, t, s_) for (rid, T, s_, _, d), t in zip(reqs, new)]
    del plan
lat = lat[3:]
print("thr=$1 ctas=$2 p50=%.2f max=%.2f" % (sorted(lat)[len(lat)//2], max(lat)), " ".join("%.1f" % x for x in lat))
PY
done
