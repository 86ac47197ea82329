import os, sys, time
sys.path.insert(0, ".")
import torch, bench, synth
from paper_2602_22593_b200 import flykv as F
from paper_2602_22593_b200.engine import KVSwitchEngine
w = synth.WORKLOADS["c2"]()
g = F.geometry(w.L, w.H, w.d, w.B, w.e)
nb, tabs = bench.pools_and_tables(w)
eng = KVSwitchEngine(g, nb, "cuda:0")
if len(sys.argv) > 1:
    for i, t in enumerate(eng.pools.tensors):
        synth.fill_hash_torch(t, i)
for s_, ids in zip(w.src, tabs):
    eng.cache.reserve(s_, ids)
reqs = [(i, T, s_, ids, d) for i, (T, s_, d, ids) in enumerate(zip(w.T, w.src, w.dst, tabs))]
st = eng.stream
burst = int(os.environ.get("BURST", "0"))
keep = []
with torch.cuda.stream(st):
    for it in range(burst):  # back-to-back switches, no host sync (like bench's device-timed region)
        plan = eng.plan(reqs)
        tables = eng.execute(plan)
        keep.append(tables)
        new = plan.dst_tables()
        reqs = [(rid, T, d, t, s_) for (rid, T, s_, _, d), t in zip(reqs, new)]
torch.cuda.synchronize()
keep.clear()
for it in range(60):
    ts = [time.perf_counter()]
    plan = eng.plan(reqs); ts.append(time.perf_counter())
    plan.upload(st); ts.append(time.perf_counter())
    F.kv_reshard(plan, -1, st); ts.append(time.perf_counter())
    tables = eng.alloc_tables(plan, range(eng.n_gpus)); ts.append(time.perf_counter())
    for gg, t in tables.items():
        F.kv_remap_block_tables(plan, gg, t.req_ptr, t.block_ids, t.meta, st)
    ts.append(time.perf_counter())
    host = {}
    with torch.cuda.stream(st):
        for gg, t in tables.items():
            n_res, n_ids = plan.resident(gg)
            host[gg] = (t.req_ptr.to("cpu", non_blocking=True), t.block_ids[:n_ids].to("cpu", non_blocking=True), t.meta[:n_res].to("cpu", non_blocking=True))
    ts.append(time.perf_counter())
    st.synchronize(); ts.append(time.perf_counter())
    new = plan.dst_tables()
    reqs = [(rid, T, d, t, s_) for (rid, T, s_, _, d), t in zip(reqs, new)]
    del plan
    ts.append(time.perf_counter())
    d = [(b - a) * 1e3 for a, b in zip(ts, ts[1:])]
    tot = (ts[-1] - ts[0]) * 1e3
    if tot > 9 or it < 2:
        print(f"it {it} total {tot:.1f}: plan {d[0]:.2f} upload {d[1]:.2f} reshard {d[2]:.2f} alloc {d[3]:.2f} remap {d[4]:.2f} d2h {d[5]:.2f} sync {d[6]:.2f} post {d[7]:.2f}")
print("done")
