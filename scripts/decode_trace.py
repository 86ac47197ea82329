"""Debug: one TP-layout decode launch of the c4 workload with the phase trace
(library built with -DFLYKV_DEC_TRACE); prints per-phase time statistics."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2602_22593_b200 import flykv as F  # noqa: E402
from paper_2602_22593_b200.engine import KVSwitchEngine  # noqa: E402
import bench  # noqa: E402

w = synth.WORKLOADS["c4"]()
g = F.geometry(w.L, w.H, w.d, w.B, w.e)
nb, tabs = bench.pools_and_tables(w)
eng = KVSwitchEngine(g, nb, "cuda:0", tp_degrees=(2, 4, 8))
for s_, ids in zip(w.src, tabs):
    eng.cache.reserve(s_, ids)
move = [(i, T, s_, ids_, d_) for i, (T, s_, ids_, d_) in enumerate(zip(w.T, w.src, tabs, w.dst))]
plan, views, host = eng.switch(move, read_back=True)
stream = torch.cuda.Stream()
gp = 0
t = views[gp]
meta = host[gp][2].numpy()
n_res = meta.shape[0]
lens = torch.as_tensor([w.T[int(i)] for i in meta[:, 0]], dtype=torch.int32, device="cuda:0")
q = torch.randn((n_res, 8, 128), device="cuda:0").to(torch.bfloat16)
out = torch.empty((n_res, 8, 128), dtype=torch.float32, device="cuda:0")
for _ in range(3):
    F.kv_paged_decode(g, eng.pools.tensors[gp][1].data_ptr(), n_res, t.req_ptr, t.block_ids, t.meta, lens, 8, q, out,
                      0.088, max(w.T), stream)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
F.kv_paged_decode(g, eng.pools.tensors[gp][1].data_ptr(), n_res, t.req_ptr, t.block_ids, t.meta, lens, 8, q, out,
                  0.088, max(w.T), stream)
e1.record(stream)
torch.cuda.synchronize()
print("launch ms", e0.elapsed_time(e1))
n = 2000
buf = (C.c_ulonglong * (8 * n))()
F._lib.kv_debug_decode_trace(buf, n)
tr = np.frombuffer(buf, dtype=np.uint64).reshape(n, 8).astype(np.int64)
units = int((tr[:, 0] > 0).sum())
tr = tr[:units]
tr = tr[tr[:, 1] > 0]          # units that ran (the last draw of every CTA finds none)
units = len(tr)
t0 = tr[:, 0].min()
print("units", units)
for k, name in ((1, "geometry"), (2, "tiles"), (3, "fold")):
    d = (tr[:, k] - tr[:, k - 1]) / 1e3
    print(f"{name:9s} us: mean {d.mean():7.2f} p50 {np.median(d):7.2f} max {d.max():7.2f}")
last = tr[:, 5] > 0
lf = (tr[last, 5] - tr[last, 4]) / 1e3
print("last-arriver fold us: mean %.2f p50 %.2f max %.2f n %d" % (lf.mean(), np.median(lf), lf.max(), int(last.sum())))
ends = np.maximum(tr[:, 3], tr[:, 5])
print("unit end - start (us) p50/p90/max:", np.percentile((ends - tr[:, 0]) / 1e3, [50, 90, 100]))
tiles_end = (tr[:, 2] - t0) / 1e3
print("tile phase end offsets (us) p10/p50/p90/max:", np.percentile(tiles_end, [10, 50, 90, 100]))
print("unit start offsets (us) p0/p50/p100:", np.percentile((tr[:, 0] - t0) / 1e3, [0, 50, 100]))
print("unit end offsets (us) p50/p100:", np.percentile((np.maximum(tr[:, 3], tr[:, 5]) - t0) / 1e3, [50, 100]))
per_cta = {}
for row in tr:
    per_cta.setdefault(int(row[7]), []).append(row)
print("CTAs with units", len(per_cta), "units per CTA: max", max(len(v) for v in per_cta.values()),
      "mean", np.mean([len(v) for v in per_cta.values()]))
first = sorted((min(r[0] for r in v) - t0) / 1e3 for v in per_cta.values())
print("CTA first-unit start (us) p0/p50/p90/p100:", np.percentile(first, [0, 50, 90, 100]))
busy = [sum((max(r[3], r[5]) - r[0]) for r in v) / 1e3 for v in per_cta.values()]
print("CTA busy time (us) p50/p100:", np.percentile(busy, [50, 100]))
