"""Kernel-variant sweep on one B200: reshard kernel time for the bench's c2
plan (idempotent until commit, so one plan is re-run), for each variant and
CTA count, next to a plain device-to-device copy of the same byte count."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402
from paper_2602_22593_b200 import flykv as F  # noqa: E402
from paper_2602_22593_b200.engine import KVSwitchEngine  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    w = synth.WORKLOADS[cfg]()
    g = F.geometry(w.L, w.H, w.d, w.B, w.e)
    nb, tabs = bench.pools_and_tables(w)
    eng = KVSwitchEngine(g, nb, "cuda:0")
    for s_, ids in zip(w.src, tabs):
        eng.cache.reserve(s_, ids)
    reqs = [(i, T, s_, ids, d) for i, (T, s_, d, ids) in enumerate(zip(w.T, w.src, w.dst, tabs))]
    if os.environ.get("REVERSE"):  # measure the backward direction: commit the forward switch first
        p_, _, _ = eng.switch(reqs, read_back=True)
        reqs = [(i, T, d, t, s_) for (i, T, s_, _, d), t in zip(reqs, p_.dst_tables())]
        del p_
    plan = eng.plan(reqs)
    st, _ = plan.stats()
    algo = (st["n_atoms"] + st["n_atom_writes"]) * st["atom_bytes"]
    stream = eng.stream
    plan.upload(stream)
    res = {"config": cfg, "algorithmic_bytes": algo}

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        evs = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        ts = sorted(x.elapsed_time(y) for x, y in evs)
        return ts[len(ts) // 2]

    combos = os.environ.get("VARIANTS", "0:1,0:2,1:1,1:2,1:3,2:0")
    for impl, ctas in [tuple(int(x) for x in c.split(":")) for c in combos.split(",")]:
        try:
            F.set_reshard_impl(impl, ctas)
            ms = timeit(lambda: F.kv_reshard(plan, -1, stream))
            key = f"impl{impl}_ctas{ctas}"
            res[key if key not in res else key + "_again"] = {"ms": ms, "GBps": algo / ms / 1e6}
        except Exception as e:  # noqa: BLE001
            res[f"impl{impl}_ctas{ctas}"] = str(e)
        print(json.dumps(res), flush=True)
    F.set_reshard_impl(0, 0)
    # comparator: the same re-layout through a staging buffer (pack, then
    # unpack) -- what pack -> all-to-all -> unpack costs in HBM alone
    stg = torch.empty(st["n_atom_slots"] * st["atom_bytes"], dtype=torch.uint8, device="cuda:0")
    ms = timeit(lambda: (F.kv_reshard_staged(plan, -1, stg, stg.numel(), 1, stream),
                         F.kv_reshard_staged(plan, -1, stg, stg.numel(), 2, stream)))
    res["staged_pack_unpack"] = {"ms": ms, "GBps_of_fused_bytes": algo / ms / 1e6}
    del stg
    # the per-destination variant (kv_pack -> identity all-to-all -> kv_unpack)
    a2a_buf = torch.empty(st["payload_bytes"], dtype=torch.uint8, device="cuda:0")
    _, mat = plan.stats()
    nn = mat.shape[0]
    flat = np.zeros(nn * nn + 1, dtype=np.int64)
    flat[1:] = np.cumsum(mat.reshape(-1))
    off = flat[:-1].reshape(nn, nn)

    def pack_unpack():
        for s_ in range(nn):
            if mat[s_].sum():
                F.kv_pack(plan, s_, a2a_buf, off[s_], stream)
        for d in range(nn):
            if mat[:, d].sum():
                F.kv_unpack(plan, d, a2a_buf, off[:, d], stream)
    ms = timeit(pack_unpack)
    res["a2a_pack_unpack"] = {"ms": ms, "GBps_of_fused_bytes": algo / ms / 1e6}

    def pack_only():
        for s_ in range(nn):
            if mat[s_].sum():
                F.kv_pack(plan, s_, a2a_buf, off[s_], stream)

    def unpack_only():
        for d in range(nn):
            if mat[:, d].sum():
                F.kv_unpack(plan, d, a2a_buf, off[:, d], stream)
    res["a2a_pack_only_ms"] = timeit(pack_only)
    res["a2a_unpack_only_ms"] = timeit(unpack_only)
    F.set_reshard_impl(2, 0)   # kv_pack through the TMA bulk ring (loads into shared memory, bulk stores into the send chunks)
    res["a2a_pack_only_tma_ms"] = timeit(pack_only)
    F.set_reshard_impl(0, 0)
    del a2a_buf
    n = st["payload_bytes"]
    a = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    with torch.cuda.stream(stream):
        ms = timeit(lambda: b.copy_(a))
    res["torch_copy_same_bytes"] = {"ms": ms, "GBps": 2 * n / ms / 1e6}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
