"""Phase breakdown of kv_switch / kv_switch_back on c4gqa1 (forward 8 replicas, reverse 1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, synth
from paper_2602_22593_b200 import flykv as F
from paper_2602_22593_b200.engine import KVSwitchEngine
cfg = sys.argv[1] if len(sys.argv) > 1 else "c4gqa1"
w = synth.WORKLOADS[cfg]()
g = F.geometry(w.L, w.H, w.d, w.B, w.e)
nb, tabs = bench.pools_and_tables(w)
eng = KVSwitchEngine(g, nb, "cuda:0")
for s_, ids in zip(w.src, tabs):
    eng.cache.reserve(s_, ids)
reqs = [(i, T, s_, ids, d) for i, (T, s_, d, ids) in enumerate(zip(w.T, w.src, w.dst, tabs))]
st = eng.stream
prev = None
for k in range(12):
    t0 = time.perf_counter()
    p = F.kv_switch(eng.cache, reqs, st) if prev is None else F.kv_switch_back(eng.cache, prev, st)
    wall = (time.perf_counter() - t0) * 1e3
    s = p.stats()[0]
    print("fwd" if k % 2 == 0 else "rev", "wall %.3f plan %.3f enq %.3f wait %.3f read %.3f h2d %d segs %d" % (
        wall, s["t_plan_ns"] / 1e6, s["t_enqueue_ns"] / 1e6, s["t_wait_ns"] / 1e6, s["t_read_ns"] / 1e6, s["h2d_bytes"], s["n_segments"]))
    prev = p
