#!/usr/bin/env python
"""Modelled N-GPU times of every BASELINE config from the product planner's
own byte matrices (CPU only, fake pool pointers: nothing is moved).

t_min = max over GPUs of max(egress / link, ingress / link, (reads + writes) / HBM)
(SURVEY 8(d)), link = 770 GB/s per direction (B200_PROFILING.md measured peer
copy), HBM = 6.65 TB/s (fallback).  t_ordered_ms: bench.ordered_link_model of
the kernels' actual work order (plan order vs the mixed order, kv_cache_set_work_order), which
charges concurrent senders that hit the same receiver.  Reported with the identity rank IDs (R3)
and with kv_suggest_rank_ids (N2).  This is a model of multi-GPU runs that
could not be measured in round 1, not a measurement.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2602_22593_b200 import flykv as F  # noqa: E402


def model(key, rank_ids="identity", reverse=False):
    w = synth.WORKLOADS[key]()
    g = F.geometry(w.L, w.H, w.d, w.B, w.e)
    nb, tabs = bench.pools_and_tables(w)
    bases = [[(1 << 44) + (r << 38) + (l << 32) for l in range(w.L)] for r in range(w.n_gpus)]
    cache = F.KVCache(g, nb, bases, (2, 4, 8))
    for s, ids in zip(w.src, tabs):
        cache.reserve(s, ids)
    reqs = [(i, T, s, ids, d, None, None) for i, (T, s, d, ids) in enumerate(zip(w.T, w.src, w.dst, tabs))]
    if rank_ids == "suggest":
        rid = {grp: F.kv_suggest_rank_ids(cache, reqs, grp) for grp in sorted(set(tuple(d) for d in w.dst)) if grp[1] > 1}
        reqs = [r[:6] + (rid.get(tuple(r[4])),) for r in reqs]
    try:
        plan = cache.plan_switch(reqs)
        waves = 1
    except F.FlyKVError:
        return {"config": key, "rank_ids": rank_ids, "error": "does not fit in one shot with the bench pool sizing"}
    if reverse:  # the bench's return switch: every request back to its source group
        new = plan.dst_tables()
        plan.commit()
        reqs = [(rid, T, d, t_, s_, drid, srid) for (rid, T, s_, _, d, srid, drid), t_ in zip(reqs, new)]
        plan = cache.plan_switch(reqs)
    st, mat = plan.stats()
    plan.destroy()
    t, eg, ing, hb = bench.nvlink_roofline(mat, bench.FALLBACK_HBM_GBS)
    ordered = {}
    for order, name in ((0, "plan_order"), (1, "mixed")):
        cache.set_work_order(order)
        p2 = cache.plan_switch(reqs)
        ordered[name] = bench.ordered_link_model([p2.work_order(x) for x in range(w.n_gpus)], bench.FALLBACK_HBM_GBS)
        p2.destroy()
    cache.set_work_order(1)
    return {"config": key, "direction": "reverse" if reverse else "forward", "workload": w.name,
            "n_gpus": w.n_gpus, "rank_ids": rank_ids, "waves": waves,
            "t_ordered_ms": {k: round(v * 1e3, 3) for k, v in ordered.items()},
            "payload_GB": round(st["payload_bytes"] / 1e9, 3), "t_min_ms": round(t * 1e3, 3),
            "max_egress_GB": round(float(eg.max()) / 1e9, 3), "max_ingress_GB": round(float(ing.max()) / 1e9, 3),
            "local_fraction": round(float(np.trace(mat) / max(mat.sum(), 1)), 4),
            "target_70pct_ms": round(t * 1e3 / 0.7, 3)}


def main():
    out = []
    for key in ("c2", "c3i", "c3ii", "c4", "c4fan", "c4gqa4", "c4gqa1", "c5"):
        for rid in ("identity", "suggest"):
            for rev in (False, True):
                r = model(key, rid, rev)
                out.append(r)
                print(json.dumps(r), flush=True)
    path = os.path.join(ROOT, "profiles", "r01_modeled_nvlink.json")
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
