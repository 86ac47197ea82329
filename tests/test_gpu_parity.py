"""GPU parity: the CUDA path (through the C ABI) against the oracle,
element by element, tolerance 0 (byte copies + integer tables, BJ).

Small cases: whole pools copied back and compared byte for byte with the C
oracle run on the same seeded host inputs; destination tables, per-GPU CSR
tables and allocator state compared exactly.  Full BASELINE size (config 2,
the bench's launch configuration): sampled atoms checked one by one against
the oracle's locate() and the content hash (synth.py), tables compared in
full with the oracle's allocator.
"""
import numpy as np
import pytest

import synth
from helpers import oracle_alloc
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _F():
    from paper_2602_22593_b200 import flykv
    return flykv


def run_parity(geo, nb, spec, seed=0, per_gpu_launch=False, check_pools=True, staged=False, a2a=False,
               work_order=1, degrees=(2, 4, 8, 16), ranges=None, one_call=False):
    """spec: list of (T, src_group, dst_group).  Runs the product on cuda:0
    (virtual ranks) and the oracle on host copies; asserts exact equality.
    work_order: the kernels' visiting order (kv_cache_set_work_order); it
    must not change any result."""
    F = _F()
    from paper_2602_22593_b200.engine import KVSwitchEngine
    og = O.Geom(*geo)
    g = F.geometry(*geo)
    eng = KVSwitchEngine(g, nb, "cuda:0", tp_degrees=degrees)
    eng.cache.set_work_order(work_order)
    for gpu, t in enumerate(eng.pools.tensors):
        synth.fill_hash_torch(t, gpu, seed=seed + 2)
    torch.cuda.synchronize()
    host_pools = [t.cpu().numpy().reshape(-1).copy() for t in eng.pools.tensors]
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    spec = [tuple(x) + (None,) * (5 - len(x)) for x in spec]  # (T, src, dst, src_rid, dst_rid)
    counts = [O.num_blocks(og, x[0], x[1][1]) for x in spec]
    w = synth.Workload("t", *geo, len(nb), [x[0] for x in spec], [x[1] for x in spec], [x[2] for x in spec])
    tabs0 = synth.source_tables(w, counts, nb, seed=seed + 1)
    oreqs, freqs = [], []
    for i, ((T, src, dst, srid, drid), ids) in enumerate(zip(spec, tabs0)):
        eng.cache.reserve(src, ids)
        for r in range(src[1]):
            held[src[0] + r][ids] = 1
        oreqs.append(O.Req(T, src, list(ids), dst, srid, drid))
        freqs.append((1000 + i, T, src, ids, dst, srid, drid))
    # GQA sources: replicas identical (R10) under the source rank IDs -- copy on both sides
    M = O.block_bytes(og)
    for (T, src, dst, srid, drid), ids in zip(spec, tabs0):
        if src[1] > og.H:
            rep = src[1] // og.H
            rid = list(srid) if srid is not None else list(range(src[1]))
            for r in range(src[1]):
                lo = src[0] + rid.index((rid[r] // rep) * rep)
                if lo == src[0] + r:
                    continue
                idx = torch.as_tensor(np.asarray(ids, dtype=np.int64), device="cuda:0")
                eng.pools.tensors[src[0] + r][:, idx] = eng.pools.tensors[lo][:, idx]
                hp = host_pools[src[0] + r].reshape(og.L, nb[src[0] + r], M)
                hp[:, ids] = host_pools[lo].reshape(og.L, nb[lo], M)[:, ids]
    plan = eng.plan(freqs)
    tables = eng.alloc_tables(plan, range(len(nb))) if (staged or per_gpu_launch) else None
    if a2a:  # pack into per-destination chunks -> (identity all-to-all) -> unpack
        tables, _ = eng.execute_pack_unpack(plan)
    elif staged:  # comparator path: pack -> staging -> unpack
        st_, _ = plan.stats()
        stg = torch.empty(max(st_["n_atom_slots"] * st_["atom_bytes"], 16), dtype=torch.uint8, device="cuda:0")
        F.kv_reshard_staged(plan, -1, stg, stg.numel(), 1, eng.stream)
        F.kv_reshard_staged(plan, -1, stg, stg.numel(), 2, eng.stream)
        for gpu, t in tables.items():
            F.kv_remap_block_tables(plan, gpu, t.req_ptr, t.block_ids, t.meta, eng.stream)
    elif per_gpu_launch:
        for gpu in range(len(nb)):
            F.kv_reshard(plan, gpu, eng.stream)
        for gpu, t in tables.items():
            F.kv_remap_block_tables(plan, gpu, t.req_ptr, t.block_ids, t.meta, eng.stream)
    elif ranges is not None:   # kv_reshard_range over a partition of the pools (processes owning several)
        tables = eng.alloc_tables(plan, range(len(nb)))
        for lo, hi in ranges:
            F.kv_reshard_range(plan, lo, hi, eng.stream)
        for gpu, t in tables.items():
            F.kv_remap_block_tables(plan, gpu, t.req_ptr, t.block_ids, t.meta, eng.stream)
    elif one_call:   # kv_switch: the plan above is discarded, the one-call API re-plans the same requests
        plan.destroy()
        plan = F.kv_switch(eng.cache, freqs, eng.stream)
        tables = {}
        for gpu in range(len(nb)):
            rp, ids_, meta_ = plan.host_tables(gpu)
            tables[gpu] = type("T", (), {"req_ptr": torch.as_tensor(rp), "block_ids": torch.as_tensor(ids_),
                                         "meta": torch.as_tensor(meta_)})
    else:  # default: one reshard launch + one packed all-pool remap launch
        tables = eng.execute(plan)
    torch.cuda.synchronize()
    st, otabs = O.switch(og, host_pools, held, oreqs)
    assert st == 0
    ftabs = plan.dst_tables()
    assert [list(a) for a in ftabs] == [list(b) for b in otabs]
    for gpu in range(len(nb)):
        assert np.array_equal(eng.cache.held_mask(gpu), held[gpu]), f"allocator state differs on {gpu}"
        rp, ids, meta = O.tables(og, gpu, oreqs, otabs)
        n_res, n_ids = plan.resident(gpu)
        t = tables[gpu]
        assert np.array_equal(t.req_ptr.cpu().numpy(), rp)
        assert np.array_equal(t.block_ids[:n_ids].cpu().numpy(), ids)
        assert np.array_equal(t.meta[:n_res].cpu().numpy(), meta)
    if check_pools:
        for gpu, t in enumerate(eng.pools.tensors):
            got = t.cpu().numpy().reshape(-1)
            bad = np.nonzero(got != host_pools[gpu])[0]
            assert bad.size == 0, f"GPU {gpu}: {bad.size} bytes differ, first at {bad[:5]}"
    return eng, plan, otabs


A2A_CASES = [(8, 1, 2), (8, 2, 1), (8, 1, 8), (8, 8, 1), (8, 2, 4), (8, 4, 2), (4, 1, 8), (4, 8, 1), (2, 4, 8),
             (1, 8, 2), (1, 1, 8), (8, 8, 8)]


@pytest.mark.parametrize("H,p0,p1", A2A_CASES)
@pytest.mark.parametrize("rank_ids", [False, True])
def test_pack_all_to_all_unpack(H, p0, p1, rank_ids):
    """kv_pack -> (all-to-all) -> kv_unpack, the per-destination send-buffer
    path, equals the oracle byte for byte: merges, splits, GQA replication,
    same-degree regroupings, permuted rank IDs on both sides."""
    geo = (3, H, 64, 16, 2)
    rng = np.random.default_rng(H * 100 + p0 * 10 + p1 + 7 * rank_ids)
    n = 8
    T = [int(x) for x in rng.integers(1, 700, size=12)]
    spec = []
    for i, t in enumerate(T):
        src = ((i * p0) % n, p0)
        dst = (((i + 1) * p1) % n, p1)
        srid = [int(x) for x in rng.permutation(p0)] if rank_ids and p0 > 1 else None
        drid = [int(x) for x in rng.permutation(p1)] if rank_ids and p1 > 1 else None
        spec.append((t, src, dst, srid, drid))
    og = O.Geom(*geo)
    nb = [0] * n
    for t, s_, d_, _, _ in spec:
        for r in range(s_[1]):
            nb[s_[0] + r] += O.num_blocks(og, t, s_[1])
        for r in range(d_[1]):
            nb[d_[0] + r] += O.num_blocks(og, t, d_[1])
    # sources are scattered over whole pools, so uniform-ID allocation (R6)
    # over 8 GPUs needs room: 3x the largest per-GPU need
    nb = [3 * max(nb) + 16] * n
    run_parity(geo, nb, spec, seed=H + p0 + p1, a2a=True)


def test_tiny_config_dp2_tp2_and_back():
    """BASELINE configs[0]: L=2, H=4, d=64, B=16, 8 x 256 tokens, DP2 -> TP2 -> DP2."""
    w = synth.tiny()
    geo = (w.L, w.H, w.d, w.B, w.e)
    nb = synth.pool_blocks(w)
    spec = list(zip(w.T, w.src, w.dst))
    run_parity(geo, nb, spec)
    # and back (fresh pools, TP2 source)
    run_parity(geo, nb, [(T, d, s) for (T, s, d) in spec], seed=5)


GRID = [(H, p0, p1) for H in (1, 2, 4, 8) for p0 in (1, 2, 4, 8) for p1 in (1, 2, 4, 8) if p0 != p1]


@pytest.mark.parametrize("work_order", [1, 0])
@pytest.mark.parametrize("H,p0,p1", GRID)
def test_grid_ragged(H, p0, p1, work_order):
    """All degree pairs up to 8 (incl. GQA replication p > H), ragged T
    spanning many blocks, partial tail atoms, 2 KiB atoms, 8 virtual ranks."""
    geo = (3, H, 64, 16, 2)
    n_gpus = 8
    Ts = [1, 15, 16, 17, 33, 100, 257, 1000, 31, 64]
    spec = [(T, ((i * p0) % n_gpus, p0), (((i + 3) * p1) % n_gpus, p1)) for i, T in enumerate(Ts)]
    nb = [256] * n_gpus
    run_parity(geo, nb, spec, seed=H * 7 + p0 + 3 * p1, work_order=work_order)


@pytest.mark.parametrize("n_gpus,H,p0,p1", [(16, 16, 1, 16), (16, 8, 1, 16), (16, 16, 8, 16), (16, 4, 16, 2),
                                             (16, 2, 4, 16), (32, 8, 1, 32), (32, 32, 4, 32), (32, 4, 32, 8),
                                             (64, 8, 1, 64), (64, 64, 64, 1)])
def test_wide_groups(n_gpus, H, p0, p1):
    """Degrees beyond one 8-GPU node (a B200 NVL72 rack is one NVLink domain
    of 72 GPUs): 16-64 virtual pools, TP16/32/64 merges and splits, with
    and without GQA replication (p > H), whole pools vs the oracle."""
    geo = (2, H, 64, 16, 2)
    Ts = [1, 17, 100, 257, 700, 64]
    spec = [(T, ((i * p0) % n_gpus, p0), (((i + 1) * p1) % n_gpus, p1)) for i, T in enumerate(Ts)]
    nb = [96] * n_gpus
    run_parity(geo, nb, spec, seed=n_gpus + H + p0 + p1, degrees=(2, 4, 8, 16, 32, 64))


@pytest.mark.parametrize("d,B,e", [(128, 16, 2), (24, 16, 2), (8, 4, 2), (256, 16, 2), (64, 16, 4), (16, 1, 2)])
def test_atom_sizes(d, B, e):
    """4 KiB (the configs), 768 B / 64 B / 32 B (generic path), 8 KiB, fp32-sized elements."""
    geo = (2, 4, d, B, e)
    spec = [(T, (i % 4, 1), (0, 4) if i % 2 else (i % 4 // 2 * 2, 2)) for i, T in enumerate([5, 130, 77, 1, 64, 200])]
    w = synth.Workload("t", *geo, 4, [s[0] for s in spec], [s[1] for s in spec], [s[2] for s in spec])
    run_parity(geo, synth.pool_blocks(w, slack=1.5), spec, seed=d + B + e)


def test_per_gpu_launches_and_mixed_plan():
    """Per-source-GPU launches (the one-process-per-GPU launch shape), a
    mixed plan with no-ops, empty requests and merges/splits together."""
    geo = (2, 8, 128, 16, 2)
    spec = [(300, (0, 1), (0, 2)), (0, (1, 1), (0, 4)), (77, (2, 2), (2, 2)), (513, (4, 4), (4, 1)),
            (129, (3, 1), (0, 8)), (1, (6, 2), (0, 4)), (64, (5, 1), (5, 1))]
    run_parity(geo, [128] * 8, spec, seed=11, per_gpu_launch=True)


@pytest.mark.parametrize("work_order", [1, 0])
@pytest.mark.parametrize("mode", ["per_gpu", "staged", "a2a", "one_launch"])
def test_mixed_order_splits(work_order, mode):
    """TP8 -> 8 x DP1 and TP4 x 2 -> DP (the splits whose senders converge on
    one receiver in plan order) with enough atoms per sender for many quanta
    of the mixed order (K > 1, holes at the buckets' ragged ends): every
    launch shape and both orders equal the oracle byte for byte."""
    geo = (8, 8, 64, 16, 2)
    rng = np.random.default_rng(31 + work_order)
    T = [int(x) for x in rng.integers(900, 2600, size=16)]
    spec = [(t, (0, 8), (i % 8, 1)) for i, t in enumerate(T[:10])]
    spec += [(t, ((i % 2) * 4, 4), ((i % 2) * 4 + (i // 2) % 4, 1)) for i, t in enumerate(T[10:])]
    run_parity(geo, [900] * 8, spec, seed=17, per_gpu_launch=mode == "per_gpu", staged=mode == "staged",
               a2a=mode == "a2a", work_order=work_order)


def test_empty_plan():
    F = _F()
    from paper_2602_22593_b200.engine import KVSwitchEngine
    eng = KVSwitchEngine(F.geometry(2, 4, 64, 16, 2), [8, 8], "cuda:0")
    plan, tables, host = eng.switch([], read_back=True)
    for g in (0, 1):
        assert plan.resident(g) == (0, 0)
        assert host[g][0].tolist() == [0]


def test_round_trip_restores_contents():
    """DP4 -> TP2x2 -> DP4 (config 2 shape, shortened): the logical KV of
    every request is back byte for byte (checked via the oracle locate)."""
    geo = (4, 8, 128, 16, 2)
    og = O.Geom(*geo)
    w = synth.llama8b_dp4_tp2x2(n_req=16)
    w.T = [t // 8 for t in w.T]
    spec = list(zip(w.T, w.src, w.dst))
    nb = synth.pool_blocks(w)
    eng, plan, tabs1 = run_parity(geo, nb, spec, seed=3)
    F = _F()
    before = [t.clone() for t in eng.pools.tensors]
    back = [(2000 + i, T, d, tabs1[i], s) for i, (T, s, d) in enumerate(spec)]
    plan2, tables2, _ = eng.switch(back, read_back=True)
    torch.cuda.synchronize()
    tabs2 = plan2.dst_tables()
    atom = og.B * og.d * og.e
    M = O.block_bytes(og)
    for i, (T, s, d) in enumerate(spec):
        for l in range(og.L):
            for kv in range(2):
                for h in range(og.H):
                    for c in range(-(-T // og.B)):
                        g1, o1 = O.locate(og, d[0], d[1], tabs1[i], kv, h, c * og.B)
                        g2, o2 = O.locate(og, s[0], s[1], tabs2[i], kv, h, c * og.B)
                        a = before[g1].view(-1)[l * nb[g1] * M + o1:][:atom]
                        b = eng.pools.tensors[g2].view(-1)[l * nb[g2] * M + o2:][:atom]
                        assert torch.equal(a, b)


@pytest.mark.slow
@pytest.mark.parametrize("cfg,n_req,frag,impl", [("c2", 0, 1.25, 0), ("c4", 0, 1.25, 0), ("c4fan", 0, 1.25, 0),
                                                 ("c4gqa4", 0, 1.25, 0),
                                                 ("c4gqa1", 0, 1.25, 0), ("c3i", 64, 1.25, 0), ("c3ii", 64, 1.25, 0),
                                                 ("c5", 0, 1.0, 0), ("single", 0, 1.25, 0),
                                                 ("c2", 0, 1.25, 2), ("c4gqa4", 0, 1.25, 2),
                                                 ("c2", 0, 1.25, "a2a"), ("c4gqa1", 0, 1.25, "a2a")])
def test_full_size_all_atoms(cfg, n_req, frag, impl):
    """Every BASELINE config at the size and in the launch configuration the
    bench times (virtual ranks on one B200, the bench's pool sizing and
    placement, one reshard launch; config 3 on the bench's 64-request prefix,
    config 4(ii) = c4fan, the single-replica fan-out, config 5 in full with
    `--frag 1.0`): destination tables equal the oracle's allocator in full,
    and EVERY BYTE of every pool (up to 158 GB) equals the oracle's expected
    pool -- every destination atom (up to 13.4M x 4 KiB, all GQA replicas)
    the content hash of the source position the oracle maps it from, every
    other byte (free blocks, released sources, tail slots past T) its
    untouched content hash, so a stray write anywhere fails.  impl 2: the TMA
    bulk-ring variant of the reshard kernel on the same checks."""
    F = _F()
    from paper_2602_22593_b200.engine import KVSwitchEngine
    F.set_reshard_impl(0 if impl == "a2a" else impl, 0)
    try:
        _full_size_all_atoms(F, KVSwitchEngine, cfg, n_req, frag, a2a=impl == "a2a")
    finally:
        F.set_reshard_impl(0, 0)


def _full_size_all_atoms(F, KVSwitchEngine, cfg, n_req, frag, a2a=False):
    w = synth.WORKLOADS[cfg]()
    if n_req:
        w = synth.Workload(w.name, w.L, w.H, w.d, w.B, w.e, w.n_gpus, w.T[:n_req], w.src[:n_req], w.dst[:n_req])
    og = O.Geom(w.L, w.H, w.d, w.B, w.e)
    n0 = [O.num_blocks(og, T, s[1]) for T, s in zip(w.T, w.src)]
    n1 = [O.num_blocks(og, T, d[1]) for T, d in zip(w.T, w.dst)]
    nb, tabs0 = synth.realistic_pools(w, n0, n1, frag=frag)
    eng = KVSwitchEngine(F.geometry(w.L, w.H, w.d, w.B, w.e), nb, "cuda:0")
    for gpu, t in enumerate(eng.pools.tensors):
        synth.fill_hash_torch(t, gpu)
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    reqs, oreqs = [], []
    for i, (T, s, d, ids) in enumerate(zip(w.T, w.src, w.dst, tabs0)):
        eng.cache.reserve(s, ids)
        for r in range(s[1]):
            held[s[0] + r][ids] = 1
        reqs.append((i, T, s, ids, d))
        oreqs.append(O.Req(T, s, list(ids), d))
    if a2a:  # pack -> all-to-all -> unpack path, then the same checks
        plan = eng.plan(reqs)
        eng.execute_pack_unpack(plan)
        rp_, ids_, meta_ = (x.cpu() for x in eng._packed)
        host = {}
        o_r = o_i = 0
        for gpu in range(w.n_gpus):
            n_res, n_ids = plan.resident(gpu)
            host[gpu] = (rp_[o_r + gpu:o_r + gpu + n_res + 1], ids_[o_i:o_i + n_ids], meta_[o_r:o_r + n_res])
            o_r += n_res
            o_i += n_ids
    else:
        plan, tables, host = eng.switch(reqs, read_back=True)
    st, otabs = O.switch(og, None, held, oreqs, copy=False)
    assert st == 0
    assert [list(a) for a in plan.dst_tables()] == [list(b) for b in otabs]
    for gpu in range(w.n_gpus):
        rp, ids, meta = O.tables(og, gpu, oreqs, otabs)
        assert np.array_equal(host[gpu][0].numpy(), rp)
        assert np.array_equal(host[gpu][1].numpy(), ids)
        assert np.array_equal(host[gpu][2].numpy(), meta)
        assert np.array_equal(eng.cache.held_mask(gpu), held[gpu])
    # Whole pools, every byte: the expected pool is the content hash
    # everywhere (untouched blocks, freed sources, tail slots past T in the
    # destination blocks, R9) with every destination atom (all replicas)
    # replaced by the hash of the source position the oracle maps it from.
    # Built and compared in chunks of 64 Mi words (atoms never straddle one).
    M = O.block_bytes(og)
    atom_words = og.B * og.d * og.e // 4
    ar = torch.arange(atom_words, dtype=torch.int64, device="cuda:0")
    per_gpu = {g: ([], [], []) for g in range(w.n_gpus)}
    n_writes = 0
    for i in range(len(w.T)):
        sg, so, dg, do = O.atom_map(og, nb, w.T[i], w.src[i], tabs0[i], w.dst[i], otabs[i])
        n_writes += dg.size
        for gd in np.unique(dg):
            m = dg == gd
            per_gpu[int(gd)][0].append(sg[m].astype(np.int64))
            per_gpu[int(gd)][1].append(so[m] // 4)
            per_gpu[int(gd)][2].append(do[m] // 4)
    assert n_writes * og.B * og.d * og.e == plan.stats()[0]["payload_bytes"]
    chunk = 64 * 2 ** 20
    assert chunk % atom_words == 0
    for gd in range(w.n_gpus):
        parts = per_gpu[gd]
        if parts[0]:
            d_w = torch.as_tensor(np.concatenate(parts[2]), device="cuda:0")
            order = torch.argsort(d_w)
            d_w = d_w[order]
            s_g = torch.as_tensor(np.concatenate(parts[0]), device="cuda:0")[order]
            s_w = torch.as_tensor(np.concatenate(parts[1]), device="cuda:0")[order]
            assert d_w.numel() == torch.unique(d_w).numel()        # every destination atom written once
        else:
            d_w = s_g = s_w = torch.zeros(0, dtype=torch.int64, device="cuda:0")
        flat = eng.pools.tensors[gd].reshape(-1).view(torch.int32)
        for w0 in range(0, flat.numel(), chunk):
            w1 = min(flat.numel(), w0 + chunk)
            exp = synth.hash32_torch(gd, torch.arange(w0, w1, dtype=torch.int64, device="cuda:0"))
            a, b = (int(x) for x in torch.searchsorted(d_w, torch.tensor([w0, w1], device="cuda:0")))
            for c0 in range(a, b, 16384):
                c1 = min(b, c0 + 16384)
                exp.view(-1, atom_words)[(d_w[c0:c1] - w0) // atom_words] = synth.hash32_torch(
                    s_g[c0:c1, None], s_w[c0:c1, None] + ar[None, :])
            same = torch.equal(flat[w0:w1], exp)
            if not same:
                bad = torch.nonzero(flat[w0:w1] != exp)[:4].flatten() + w0
                raise AssertionError(f"pool {gd}: words differ from the oracle's expected pool at {bad.tolist()}")
            del exp


def test_weight_views_gather():
    """Eq.1 views on a device matrix, materialised by the gather kernel, equal
    the numpy oracle slices (bit exact)."""
    F = _F()
    from oracle import weights as W
    Hq, Hkv, d, hidden = 16, 4, 32, 96
    rows = (Hq + 2 * Hkv) * d
    full = torch.randn(rows, hidden, device="cuda:0").to(torch.bfloat16)
    host = full.view(torch.int16).cpu().numpy()
    for m in (1, 2, 4, 8):
        for r in range(m):
            v = F.weight_shard_view(F.weight_desc(full, rows, hidden, 2, F.KV_W_QKV, num_q_heads=Hq,
                                                  num_kv_heads=Hkv, head_dim=d), r, m)
            nrow = sum(s.rows for s in v.segments())
            out = torch.empty(nrow, hidden, dtype=torch.bfloat16, device="cuda:0")
            F.kv_gather_view(v, out)
            ref = np.concatenate(W.view_qkv(host, r, m, Hq, Hkv, d))
            torch.cuda.synchronize()
            assert np.array_equal(out.view(torch.int16).cpu().numpy(), ref)
            v = F.weight_shard_view(F.weight_desc(full, rows, hidden, 2, F.KV_W_ROW), r, m)
            out = torch.empty(rows, hidden // m, dtype=torch.bfloat16, device="cuda:0")
            F.kv_gather_view(v, out)
            torch.cuda.synchronize()
            (ref,) = W.view_row(host, r, m)
            assert np.array_equal(out.view(torch.int16).cpu().numpy(), ref)


def test_launch_counter_moves():
    F = _F()
    before = F.launch_count()
    test_empty_plan()
    geo = (1, 2, 64, 16, 2)
    run_parity(geo, [16, 16], [(40, (0, 1), (0, 2))])
    assert F.launch_count() >= before + 3


@pytest.mark.parametrize("a2a", [False, True])
@pytest.mark.parametrize("impl", [1, 2, 3])
@pytest.mark.parametrize("H,p0,p1", [(8, 1, 2), (8, 2, 1), (4, 1, 8), (2, 8, 1), (8, 4, 8)])
@pytest.mark.parametrize("d", [64, 128])
def test_reshard_variants(impl, H, p0, p1, d, a2a):
    """Every reshard kernel variant (LDG/STG, TMA bulk ring, 2 atoms in
    flight) is bit-exact, incl. GQA replication, 2 KiB and 4 KiB atoms; with
    a2a, the same variants as kv_pack into per-destination send chunks (TMA
    bulk stores into the contiguous send buffer under impl 2)."""
    F = _F()
    F.set_reshard_impl(impl, 0)
    try:
        geo = (2, H, d, 16, 2)
        Ts = [1, 15, 16, 17, 33, 100, 257, 1000, 31, 64, 700, 2049]
        spec = [(T, ((i * p0) % 8, p0), (((i + 3) * p1) % 8, p1)) for i, T in enumerate(Ts)]
        run_parity(geo, [400] * 8, spec, seed=impl * 31 + H + p0 + p1, a2a=a2a)
    finally:
        F.set_reshard_impl(0, 0)


@pytest.mark.parametrize("one_call", [False, True, "schedule"])
def test_memory_bounded_waves_gpu(one_call):
    """SURVEY 8(f) N1 on the device: a promotion that does not fit in one
    shot runs in waves (kv_plan_waves -> switch per wave, or every wave in
    one kv_switch_multi call with no sync between waves); whole pools equal
    the oracle applied wave after wave."""
    F = _F()
    from paper_2602_22593_b200.engine import KVSwitchEngine
    geo = (2, 8, 64, 16, 2)
    og = O.Geom(*geo)
    nb = [56] * 8
    eng = KVSwitchEngine(F.geometry(*geo), nb, "cuda:0")
    for gpu, t in enumerate(eng.pools.tensors):
        synth.fill_hash_torch(t, gpu, seed=77)
    torch.cuda.synchronize()
    host = [t.cpu().numpy().reshape(-1).copy() for t in eng.pools.tensors]
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    rng = np.random.default_rng(9)
    reqs = []
    for i in range(24):
        T = int(rng.integers(80, 200))
        src = (i % 8, 1)
        ids = oracle_alloc(eng.cache, held, src, O.num_blocks(og, T, 1))
        reqs.append((i, T, src, ids, (0, 8)))
    with pytest.raises(F.FlyKVError):
        eng.plan(reqs)
    waves = F.kv_plan_waves(eng.cache, reqs)
    assert len(waves) > 1
    if one_call == "schedule":  # kv_switch_waves: the same schedule and every wave in one call
        wv, plans = F.kv_switch_waves(eng.cache, reqs, split=False, stream=eng.stream)
        assert wv == [[(i, 0, reqs[i][1]) for i in range(a, b)] for a, b in waves]
        out = [(p, None, None) for p in plans]
    elif one_call:
        out = [(p, None, None) for p in F.kv_switch_multi(eng.cache, [reqs[a:b] for a, b in waves], eng.stream)]
        torch.cuda.synchronize()
    else:
        out = eng.switch_waves(reqs, read_back=True)
    assert len(out) == len(waves)
    for (a, b), (plan, tables, hb) in zip(waves, out):
        if one_call:  # the tables kv_switch_multi read back equal the plan's
            for gpu in range(len(nb)):
                rp, ids_, meta = plan.host_tables(gpu)
                orp, oids, ometa = O.tables(og, gpu, [O.Req(T, s, list(ids), d) for (_, T, s, ids, d) in reqs[a:b]],
                                            [list(x) for x in plan.dst_tables()])
                assert np.array_equal(rp, orp) and np.array_equal(ids_, oids) and np.array_equal(meta, ometa)
        st, otabs = O.switch(og, host, held, [O.Req(T, s, list(ids), d) for (_, T, s, ids, d) in reqs[a:b]])
        assert st == 0
        assert [list(x) for x in plan.dst_tables()] == [list(y) for y in otabs]
    for gpu, t in enumerate(eng.pools.tensors):
        assert np.array_equal(t.cpu().numpy().reshape(-1), host[gpu])
        assert np.array_equal(eng.cache.held_mask(gpu), held[gpu])


def test_failed_wave_keeps_committed_waves():
    """kv_switch_multi whose second wave does not fit (OUT_OF_BLOCKS): the
    first wave has committed (its sources are released), so the error hands
    its plan over with its tables read back -- tables, pools and
    allocator equal the oracle after wave 0 alone; the failing wave changed
    nothing."""
    F = _F()
    from paper_2602_22593_b200.engine import KVSwitchEngine
    geo = (2, 8, 64, 16, 2)
    og = O.Geom(*geo)
    nb = [56] * 8
    eng = KVSwitchEngine(F.geometry(*geo), nb, "cuda:0")
    for gpu, t in enumerate(eng.pools.tensors):
        synth.fill_hash_torch(t, gpu, seed=78)
    torch.cuda.synchronize()
    host = [t.cpu().numpy().reshape(-1).copy() for t in eng.pools.tensors]
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    rng = np.random.default_rng(10)
    reqs = []
    for i in range(24):
        T = int(rng.integers(80, 200))
        src = (i % 8, 1)
        reqs.append((i, T, src, oracle_alloc(eng.cache, held, src, O.num_blocks(og, T, 1)), (0, 8)))
    (a, b) = F.kv_plan_waves(eng.cache, reqs)[0]
    with pytest.raises(F.FlyKVError) as e:
        F.kv_switch_multi(eng.cache, [reqs[a:b], reqs[b:]], eng.stream)
    assert e.value.name == "KV_ERR_OUT_OF_BLOCKS" and len(e.value.plans) == 1
    plan = e.value.plans[0]
    oreqs = [O.Req(T, s, list(ids), d) for (_, T, s, ids, d) in reqs[a:b]]
    st, otabs = O.switch(og, host, held, oreqs)
    assert st == 0
    assert [list(x) for x in plan.dst_tables()] == [list(y) for y in otabs]
    for gpu in range(len(nb)):
        rp, ids_, meta = plan.host_tables(gpu)
        orp, oids, ometa = O.tables(og, gpu, oreqs, otabs)
        assert np.array_equal(rp, orp) and np.array_equal(ids_, oids) and np.array_equal(meta, ometa)
        assert np.array_equal(eng.cache.held_mask(gpu), held[gpu])
        assert np.array_equal(eng.pools.tensors[gpu].cpu().numpy().reshape(-1), host[gpu])


@pytest.mark.parametrize("seed", range(10))
def test_random_mixed_plans(seed):
    """Randomised plans: random H, head_dim, degrees (merge, split, lateral,
    no-op), lengths incl. 0, 8 virtual ranks; bit-exact against the oracle."""
    rng = np.random.default_rng(1000 + seed)
    H = int(rng.choice([1, 2, 4, 8]))
    d = int(rng.choice([64, 128]))
    geo = (int(rng.integers(1, 4)), H, d, 16, 2)
    n_gpus = 8
    spec = []
    used_src = set()
    for i in range(int(rng.integers(1, 14))):
        p0 = int(rng.choice([1, 2, 4, 8]))
        p1 = int(rng.choice([1, 2, 4, 8]))
        g0 = int(rng.integers(0, n_gpus // p0)) * p0
        g1 = int(rng.integers(0, n_gpus // p1)) * p1
        T = int(rng.choice([0, 1, int(rng.integers(2, 40)), int(rng.integers(40, 900))]))
        spec.append((T, (g0, p0), (g1, p1)))
    run_parity(geo, [480] * n_gpus, spec, seed=seed)


def test_weight_view_contiguous_alias():
    """the TP-rank view of the fused W^QKV is contiguous in virtual
    memory but maps the DP replica's physical memory (CUDA VMM alias, 0 bytes
    copied).  Llama-3-70B-shaped QKV (64 q heads, 8 kv heads, d=128,
    hidden 8192, bf16) at TP2/4/8: the alias reads back exactly the oracle's
    Eq.1 slices, and a write through the DP address is visible through it."""
    F = _F()
    from oracle import weights as W
    Hq, Hkv, d, hidden = 64, 8, 128, 8192
    rows = (Hq + 2 * Hkv) * d
    g = F.vmm_granularity(0)
    assert g <= 2 * 2 ** 20
    full = torch.randn(rows, hidden, device="cuda:0").to(torch.bfloat16)
    host = full.view(torch.int16).cpu().numpy()
    buf = F.VmmBuffer(rows * hidden * 2)
    F.kv_gather_view(F.weight_shard_view(F.weight_desc(full, rows, hidden, 2, F.KV_W_COLUMN), 0, 1), buf.ptr)
    torch.cuda.synchronize()
    for m in (2, 4, 8):
        for r in (0, m - 1):
            v = F.weight_shard_view(F.weight_desc(buf.ptr, rows, hidden, 2, F.KV_W_QKV, num_q_heads=Hq,
                                                  num_kv_heads=Hkv, head_dim=d), r, m)
            ptr, nbytes = F.weight_view_alias(buf, v)
            nrow = nbytes // (2 * hidden)
            out = torch.empty(nrow, hidden, dtype=torch.bfloat16, device="cuda:0")
            F.kv_gather_view(F.weight_shard_view(F.weight_desc(ptr, nrow, hidden, 2, F.KV_W_COLUMN), 0, 1), out)
            torch.cuda.synchronize()
            ref = np.concatenate(W.view_qkv(host, r, m, Hq, Hkv, d))
            assert np.array_equal(out.view(torch.int16).cpu().numpy(), ref)
            if m == 8 and r == m - 1:
                # write-through: overwrite the DP replica's K rows of this rank's head
                new = torch.full((d, hidden), 3.0, dtype=torch.bfloat16, device="cuda:0")
                kseg = v.seg[1]
                F.kv_gather_view(F.weight_shard_view(F.weight_desc(new, d, hidden, 2, F.KV_W_COLUMN), 0, 1), kseg.ptr)
                F.kv_gather_view(F.weight_shard_view(F.weight_desc(ptr, nrow, hidden, 2, F.KV_W_COLUMN), 0, 1), out)
                torch.cuda.synchronize()
                q_rows = v.seg[0].rows
                assert torch.equal(out[q_rows:q_rows + d], new)
            F.weight_view_unalias(ptr, nbytes)
    # a view whose K/V segments are not granularity-aligned cannot be aliased
    small = F.VmmBuffer((8 + 2 * 2) * 64 * 256 * 2)
    v = F.weight_shard_view(F.weight_desc(small.ptr, (8 + 4) * 64, 256, 2, F.KV_W_QKV, num_q_heads=8, num_kv_heads=2,
                                          head_dim=64), 0, 2)
    with pytest.raises(F.FlyKVError) as e:
        F.weight_view_alias(small, v)
    assert e.value.name == "KV_ERR_INDIVISIBLE_EXTENT"
    row = F.weight_shard_view(F.weight_desc(buf.ptr, rows, hidden, 2, F.KV_W_ROW), 0, 2)
    with pytest.raises(F.FlyKVError):
        F.weight_view_alias(buf, row)
    small.close()
    buf.close()


@pytest.mark.parametrize("H,p0,p1", [(8, 1, 2), (4, 1, 8), (8, 4, 1)])
def test_staged_comparator_matches(H, p0, p1):
    """The bench comparator (pack -> staging -> unpack) produces the same bytes."""
    geo = (2, H, 128, 16, 2)
    Ts = [1, 17, 100, 257, 1000, 64]
    spec = [(T, ((i * p0) % 8, p0), (((i + 3) * p1) % 8, p1)) for i, T in enumerate(Ts)]
    run_parity(geo, [300] * 8, spec, seed=H + p0 + p1, staged=True)


def test_million_token_request():
    """One 1,048,581-token request DP -> TP8 (65,537 chunks, ragged tail):
    every destination atom checked against the oracle's atom map."""
    F = _F()
    from paper_2602_22593_b200.engine import KVSwitchEngine
    geo = (1, 8, 64, 16, 2)
    og = O.Geom(*geo)
    T = (1 << 20) + 5
    n0 = O.num_blocks(og, T, 1)
    n1 = O.num_blocks(og, T, 8)
    nb = [n0 + n1 + 64] * 8  # uniform IDs across the TP8 group (R6): equal ID ranges
    eng = KVSwitchEngine(F.geometry(*geo), nb, "cuda:0")
    for gpu, t in enumerate(eng.pools.tensors):
        synth.fill_hash_torch(t, gpu, seed=5)
    ids = np.arange(n0, dtype=np.int32)  # an oracle-side table, registered with kv_reserve
    eng.cache.reserve((0, 1), ids)
    plan, tables, host = eng.switch([(0, T, (0, 1), ids, (0, 8))], read_back=True)
    tab1 = plan.dst_tables()[0]
    sg, so, dg, do = O.atom_map(og, nb, T, (0, 1), ids, (0, 8), tab1)
    atom_words = og.B * og.d * og.e // 4
    ar = torch.arange(atom_words, dtype=torch.int64, device="cuda:0")
    flat = [t.reshape(-1).view(torch.int32) for t in eng.pools.tensors]
    for gd in range(8):
        m = dg == gd
        s_w = torch.as_tensor(so[m] // 4, device="cuda:0")
        d_w = torch.as_tensor(do[m] // 4, device="cuda:0")
        for c0 in range(0, s_w.numel(), 32768):
            sl = slice(c0, c0 + 32768)
            want = synth.hash32_torch(0, s_w[sl, None] + ar[None, :], seed=5)
            assert torch.equal(flat[gd][d_w[sl, None] + ar[None, :]], want)
    assert host[0][2].tolist() == [[0, 128, 1, 0]]


def test_many_small_requests_remap_tiles():
    """5,000 requests (1..40 tokens) DP8 -> TP8: the remap kernel's
    1024-request tiles and carries, whole pools and CSR tables vs the oracle."""
    rng = np.random.default_rng(21)
    geo = (1, 8, 64, 16, 2)
    spec = [(int(rng.integers(1, 41)), (i % 8, 1), (0, 8)) for i in range(5000)]
    run_parity(geo, [20000] * 8, spec, seed=21)


@pytest.mark.parametrize("H,p0,p1", [(8, 4, 8), (8, 2, 8), (8, 8, 4), (4, 8, 8), (2, 4, 8), (8, 1, 4), (8, 4, 4)])
def test_rank_ids_parity(H, p0, p1):
    """Rank-ID assignments on both sides (N2) incl. GQA replication and
    same-group re-permutation: whole pools, tables and first heads equal the
    oracle."""
    rng = np.random.default_rng(H * 31 + p0 * 5 + p1)
    geo = (2, H, 64, 16, 2)
    spec = []
    for i, T in enumerate([1, 17, 100, 257, 1000, 33]):
        src = ((i * p0) % 8, p0)
        dst = (((i + 1) * p1) % 8, p1)
        srid = [int(x) for x in rng.permutation(p0)]
        drid = [int(x) for x in rng.permutation(p1)]
        spec.append((T, src, dst, srid, drid))
    run_parity(geo, [400] * 8, spec, seed=H + p0 + p1)


@pytest.mark.parametrize("H,p0,p1", [(8, 1, 2), (8, 2, 1), (4, 1, 8), (8, 4, 8)])
def test_kv_switch_one_call(H, p0, p1):
    """kv_switch (plan, upload, reshard, remap, read-back, sync in one C call)
    leaves the same pools, allocator state and tables as the oracle; its
    device tables equal its host tables; kv_switch_back of it equals the
    oracle's inverse switch."""
    F = _F()
    from paper_2602_22593_b200.engine import KVSwitchEngine
    geo = (2, H, 64, 16, 2)
    og = O.Geom(*geo)
    n = 8
    rng = np.random.default_rng(H + p0 + p1)
    T = [int(x) for x in rng.integers(1, 500, size=10)]
    spec = [(t, ((i * p0) % n, p0), (((i + 1) * p1) % n, p1)) for i, t in enumerate(T)]
    nb = [0] * n
    for t, s_, d_ in spec:
        for r in range(s_[1]):
            nb[s_[0] + r] += O.num_blocks(og, t, s_[1])
        for r in range(d_[1]):
            nb[d_[0] + r] += O.num_blocks(og, t, d_[1])
    nb = [3 * max(nb) + 16] * n
    eng = KVSwitchEngine(F.geometry(*geo), nb, "cuda:0")
    for gpu, t in enumerate(eng.pools.tensors):
        synth.fill_hash_torch(t, gpu, seed=3)
    torch.cuda.synchronize()
    host_pools = [t.cpu().numpy().reshape(-1).copy() for t in eng.pools.tensors]
    w = synth.Workload("t", *geo, n, T, [x[1] for x in spec], [x[2] for x in spec])
    tabs0 = synth.source_tables(w, [O.num_blocks(og, t, s_[1]) for t, s_, _ in spec], nb, seed=4)
    held = [np.zeros(k, dtype=np.uint8) for k in nb]
    oreqs, freqs = [], []
    for i, ((t, s_, d_), ids) in enumerate(zip(spec, tabs0)):
        eng.cache.reserve(s_, ids)
        for r in range(s_[1]):
            held[s_[0] + r][ids] = 1
        oreqs.append(O.Req(t, s_, list(ids), d_))
        freqs.append((i, t, s_, ids, d_))
    if p0 > H:  # replicated sources identical (R10)
        M = O.block_bytes(og)
        for (t, s_, _), ids in zip(spec, tabs0):
            for r in range(1, s_[1]):
                lo = s_[0] + (r // (p0 // H)) * (p0 // H)
                if lo != s_[0] + r:
                    idx = torch.as_tensor(np.asarray(ids, dtype=np.int64), device="cuda:0")
                    eng.pools.tensors[s_[0] + r][:, idx] = eng.pools.tensors[lo][:, idx]
                    hp = host_pools[s_[0] + r].reshape(og.L, nb[0], M)
                    hp[:, ids] = host_pools[lo].reshape(og.L, nb[0], M)[:, ids]
    plan = F.kv_switch(eng.cache, freqs, eng.stream)
    st, otabs = O.switch(og, host_pools, held, oreqs)
    assert st == 0
    assert [list(a) for a in plan.dst_tables()] == [list(b) for b in otabs]
    for gpu in range(n):
        assert np.array_equal(eng.cache.held_mask(gpu), held[gpu])
        rp, ids, meta = O.tables(og, gpu, oreqs, otabs)
        hrp, hids, hmeta = plan.host_tables(gpu)
        assert np.array_equal(hrp, rp) and np.array_equal(hids, ids) and np.array_equal(hmeta, meta)
        drp, dids, dmeta, n_res, n_ids = plan.device_tables(gpu)
        got = torch.zeros(n_res + 1 + n_ids + 4 * n_res, dtype=torch.int32, device="cuda:0")
        for ptr, k, o in ((drp, n_res + 1, 0), (dids, n_ids, n_res + 1), (dmeta, 4 * n_res, n_res + 1 + n_ids)):
            if k:  # device-to-device copy of k int32 through a one-row view (gather kernel)
                v = F.View()
                v.n_seg, v.elem_bytes = 1, 4
                v.seg[0].ptr, v.seg[0].rows, v.seg[0].cols, v.seg[0].ld = ptr, 1, k, k
                F.kv_gather_view(v, got.data_ptr() + 4 * o)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), np.concatenate([hrp, hids, hmeta.reshape(-1)]))
    for gpu, t in enumerate(eng.pools.tensors):
        assert np.array_equal(t.cpu().numpy().reshape(-1), host_pools[gpu]), f"pool {gpu} differs"
    # and back: kv_switch_back builds the inverse requests inside the library
    back = F.kv_switch_back(eng.cache, plan, eng.stream)
    oback = [O.Req(t, d_, list(tab), s_) for (t, s_, d_), tab in zip(spec, otabs)]
    st, otabs2 = O.switch(og, host_pools, held, oback)
    assert st == 0
    assert [list(a) for a in back.dst_tables()] == [list(b) for b in otabs2]
    for gpu in range(n):
        assert np.array_equal(eng.cache.held_mask(gpu), held[gpu])
        rp, ids, meta = O.tables(og, gpu, oback, otabs2)
        hrp, hids, hmeta = back.host_tables(gpu)
        assert np.array_equal(hrp, rp) and np.array_equal(hids, ids) and np.array_equal(hmeta, meta)
    for gpu, t in enumerate(eng.pools.tensors):
        assert np.array_equal(t.cpu().numpy().reshape(-1), host_pools[gpu]), f"pool {gpu} differs after switch back"


def test_weight_switches_allocate_nothing():
    """S:152 / P:297 'no tensor movement': 1,000 DP<->TP weight-mode switches
    (Eq.1 views of a Llama-3-70B-shaped W^QKV at degrees 1/2/4/8, each also
    aliased contiguously over the replica's physical memory and released)
    allocate no device memory: torch's allocator and the driver's free-memory
    count are unchanged afterwards."""
    F = _F()
    Hq, Hkv, d, hidden = 64, 8, 128, 8192
    rows = (Hq + 2 * Hkv) * d
    buf = F.VmmBuffer(rows * hidden * 2)
    torch.cuda.synchronize()
    alloc0 = torch.cuda.memory_allocated()
    free0, _ = torch.cuda.mem_get_info()
    degrees = [1, 2, 4, 8]
    for k in range(1000):
        m = degrees[k % 4]
        r = (k // 4) % m
        v = F.weight_shard_view(F.weight_desc(buf.ptr, rows, hidden, 2, F.KV_W_QKV, num_q_heads=Hq, num_kv_heads=Hkv,
                                              head_dim=d), r, m)
        assert sum(s.rows for s in v.segments()) * hidden * 2 <= rows * hidden * 2
        ptr, nbytes = F.weight_view_alias(buf, v)
        F.weight_view_unalias(ptr, nbytes)
    torch.cuda.synchronize()
    free1, _ = torch.cuda.mem_get_info()
    assert torch.cuda.memory_allocated() == alloc0
    assert abs(free1 - free0) < 4 * 2 ** 20, (free0, free1)   # driver bookkeeping only: one TP8 view copy is 21 MB
    buf.close()


@pytest.mark.parametrize("T,src,dst,H", [(66 * 16 + 5, (0, 4), (0, 8), 8), (2000, (0, 1), (0, 8), 8),
                                         (700, (0, 2), (0, 8), 2)])
def test_long_request_promoted_in_pieces(T, src, dst, H):
    """R20 / Use Case 3: one long request whose source and destination cannot
    coexist is promoted in block-aligned token pieces over waves
    (kv_plan_pieces + one kv_switch per wave).  The pools equal the oracle's
    after the same waves, and -- the property that makes pieces legal -- the
    concatenated table is the whole request's layout at the destination
    degree: every atom (all GQA replicas) the oracle's atom map sends from the
    original source table holds the original bytes."""
    F = _F()
    from paper_2602_22593_b200.engine import KVSwitchEngine
    geo = (2, H, 64, 16, 2)
    og = O.Geom(*geo)
    n0, n1 = O.num_blocks(og, T, src[1]), O.num_blocks(og, T, dst[1])
    nb = [n0 + n1 - 1] * 8                # one block short of holding source and destination side by side
    eng = KVSwitchEngine(F.geometry(*geo), nb, "cuda:0")
    for gpu, t in enumerate(eng.pools.tensors):
        synth.fill_hash_torch(t, gpu, seed=11)
    held = [np.zeros(k, dtype=np.uint8) for k in nb]
    ids = oracle_alloc(eng.cache, held, src, n0)
    M = O.block_bytes(og)
    if src[1] > H:  # replicated source heads identical (R10)
        rep = src[1] // H
        idx = torch.as_tensor(ids.astype(np.int64), device="cuda:0")
        for r in range(src[1]):
            if r % rep:
                eng.pools.tensors[src[0] + r][:, idx] = eng.pools.tensors[src[0] + r - r % rep][:, idx]
    torch.cuda.synchronize()
    host = [t.cpu().numpy().reshape(-1).copy() for t in eng.pools.tensors]
    orig = [h.copy() for h in host]
    reqs = [(0, T, src, ids, dst)]
    with pytest.raises(F.FlyKVError):
        eng.cache.plan_switch(reqs)
    final, plans = eng.switch_pieces(reqs)
    assert len(plans) >= 2
    # replay the same pieces (one per wave: a single request) on the oracle
    parts = []
    t0 = 0
    for plan in plans:
        tab = plan.dst_tables()[0]
        t1 = min(T, t0 + len(tab) * O.block_tokens(og, dst[1]))
        b0 = O.block_tokens(og, src[1])
        piece = O.Req(t1 - t0, src, list(ids[t0 // b0: -(-t1 // b0)]), dst)
        st, otabs = O.switch(og, host, held, [piece])
        assert st == 0 and list(otabs[0]) == list(tab)
        parts.append(tab)
        t0 = t1
    assert t0 == T
    assert list(np.concatenate(parts)) == list(final[0])
    for gpu, t in enumerate(eng.pools.tensors):
        assert np.array_equal(t.cpu().numpy().reshape(-1), host[gpu]), f"pool {gpu} differs"
        assert np.array_equal(eng.cache.held_mask(gpu), held[gpu])
    # whole-request layout: original source bytes at every destination atom of the concatenated table
    sg, so, dg, do = O.atom_map(og, nb, T, src, list(ids), dst, list(final[0]))
    atom = og.B * og.d * og.e
    for k in range(0, len(sg), 97):
        a = orig[int(sg[k])][int(so[k]):int(so[k]) + atom]
        b = eng.pools.tensors[int(dg[k])].reshape(-1)[int(do[k]):int(do[k]) + atom].cpu().numpy()
        assert np.array_equal(a, b), f"atom {k}"


def test_strict_replica_mode():
    """R10 strict mode.  Sources at TP8 with H_kv = 2 hold every head on 4
    ranks (Eq.3 replication); only the canonical (lowest-owner)
    replica is read.  kv_verify_replicas finds a corrupted valid byte in a
    non-canonical replica (and decodes where), ignores stale tail slots past
    T (R9), and in strict mode kv_switch refuses the switch with no state
    change and no byte moved; once the replica is repaired the switch runs
    and matches the oracle."""
    F = _F()
    from paper_2602_22593_b200.engine import KVSwitchEngine
    geo = (2, 2, 64, 16, 2)
    og = O.Geom(*geo)
    L, H, d, B, e = geo
    nb = [48] * 8
    eng = KVSwitchEngine(F.geometry(*geo), nb, "cuda:0")
    for gpu, t in enumerate(eng.pools.tensors):
        synth.fill_hash_torch(t, gpu, seed=91)
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    reqs = []
    for i, T in enumerate((37, 64, 100)):
        ids = oracle_alloc(eng.cache, held, (0, 8), O.num_blocks(og, T, 8))
        idx = torch.as_tensor(np.asarray(ids, dtype=np.int64), device="cuda:0")
        for h in range(H):   # the 3 other replicas of head h = copies of rank 4h (R10)
            for j in range(1, 4):
                eng.pools.tensors[4 * h + j][:, idx] = eng.pools.tensors[4 * h][:, idx]
        reqs.append((i, T, (0, 8), ids, (i, 1)))
    torch.cuda.synchronize()
    plan = eng.plan(reqs)
    assert F.kv_verify_replicas(plan, eng.stream) == (0, None)
    plan.destroy()
    M = O.block_bytes(og)
    k0 = H          # chunks per source block at TP8 (B(8) = H * B)
    blk = int(reqs[0][3][2 // k0])                      # request 0 (T = 37): chunk 2 holds tokens 32..36
    base = blk * M + (2 % k0) * B * d * e               # layer 0, K half, head 0 (H_loc = 1), chunk 2
    pool1 = eng.pools.tensors[1].view(-1)               # replica j = 1 of head 0
    pool1[base + 6 * d * e] ^= 0xFF                     # token 38: stale tail slot, not compared
    plan = eng.plan(reqs)
    assert F.kv_verify_replicas(plan, eng.stream) == (0, None)
    plan.destroy()
    pool1[base + 3 * d * e + 5] ^= 0x01                 # token 35: valid
    plan = eng.plan(reqs)
    assert F.kv_verify_replicas(plan, eng.stream) == (1, 2)   # item 0 (req 0, head 0, replica 1), l 0, K, chunk 2
    plan.destroy()
    eng.cache.set_strict(True)
    before = [t.clone() for t in eng.pools.tensors]
    masks = [eng.cache.held_mask(g).copy() for g in range(8)]
    with pytest.raises(F.FlyKVError) as err:
        F.kv_switch(eng.cache, reqs, eng.stream)
    assert err.value.name == "KV_ERR_REPLICA_MISMATCH" and err.value.plans == []
    called = []   # the one-process-per-GPU calls refuse it too, before the push and the barrier
    for bar in (None, lambda: called.append(1)):
        with pytest.raises(F.FlyKVError) as err:
            F.kv_switch_range(eng.cache, reqs, 0, 8, bar, eng.stream)
        assert err.value.name == "KV_ERR_REPLICA_MISMATCH" and err.value.plans == []
    assert not called
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(before, eng.pools.tensors))
    assert all(np.array_equal(eng.cache.held_mask(g), masks[g]) for g in range(8))
    pool1[base + 3 * d * e + 5] ^= 0x01                 # repaired
    plan = F.kv_switch(eng.cache, reqs, eng.stream)
    st, otabs = O.switch(og, None, held, [O.Req(T, s, list(ids), dd) for (_, T, s, ids, dd) in reqs], copy=False)
    assert st == 0 and [list(a) for a in plan.dst_tables()] == [list(b) for b in otabs]
    for i, (_, T, s, ids, dd) in enumerate(reqs):      # every destination token equals the canonical source
        for l in range(L):
            for kv in range(2):
                for h in range(H):
                    for c in range(-(-T // B)):
                        g0, o0 = O.locate(og, 0, 8, list(ids), kv, h, c * B)
                        g1, o1 = O.locate(og, dd[0], 1, list(otabs[i]), kv, h, c * B)
                        n = min(B, T - c * B) * d * e
                        a = before[g0].view(-1)[l * nb[g0] * M + o0:][:n]
                        b = eng.pools.tensors[g1].view(-1)[l * nb[g1] * M + o1:][:n]
                        assert torch.equal(a, b)


@pytest.mark.parametrize("H,teams", [(1, [(0, 8)]), (2, [(4, 4)]), (4, [(2, 2), (6, 2)])])
def test_multicast_team_addressing_emulated(H, teams):
    """NVLS team stores (N2) without NVLS hardware: kv_cache_set_multicast in
    emulation mode (2) registers each team's replica-0 layer bases as
    ordinary pointers, so the kernel writes an atom whose replicas are a
    registered team once, to the team's first pool, and skips the other
    replicas (which the multicast fabric would deliver).  DP8 -> TP8 with
    H_kv < 8: registered teams' first pools equal the oracle, their other
    members stay untouched; unregistered teams get every replica."""
    F = _F()
    from paper_2602_22593_b200.engine import KVSwitchEngine
    geo = (2, H, 128, 16, 2)
    og = O.Geom(*geo)
    nb = [320] * 8
    eng = KVSwitchEngine(F.geometry(*geo), nb, "cuda:0")
    for gpu, t in enumerate(eng.pools.tensors):
        synth.fill_hash_torch(t, gpu, seed=55)
    torch.cuda.synchronize()
    host = [t.cpu().numpy().reshape(-1).copy() for t in eng.pools.tensors]
    before = [h.copy() for h in host]
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    rng = np.random.default_rng(H)
    reqs, oreqs = [], []
    for i in range(12):
        T = int(rng.integers(1, 300))
        src = (i % 8, 1)
        ids = oracle_alloc(eng.cache, held, src, O.num_blocks(og, T, 1))
        reqs.append((i, T, src, ids, (0, 8)))
        oreqs.append(O.Req(T, src, list(ids), (0, 8)))
    bases = eng.pools.layer_base()
    for t0, r in teams:
        eng.cache.set_multicast((t0, r), bases[t0], mode=2)
    plan = eng.plan(reqs)
    F.kv_reshard(plan, -1, eng.stream)
    torch.cuda.synchronize()
    st, otabs = O.switch(og, host, held, oreqs)
    assert st == 0 and [list(a) for a in plan.dst_tables()] == [list(b) for b in otabs]
    skipped = {t0 + j for t0, r in teams for j in range(1, r)}
    for g in range(8):
        got = eng.pools.tensors[g].cpu().numpy().reshape(-1)
        want = before[g] if g in skipped else host[g]
        assert np.array_equal(got, want), f"pool {g}"
    with pytest.raises(F.FlyKVError):
        eng.cache.set_multicast((1, 2), bases[1], mode=2)      # not aligned
    with pytest.raises(F.FlyKVError):
        eng.cache.set_multicast((0, 2), bases[0], mode=1)      # one mode per cache


def test_nvls_capability_report():
    """kv_mc_supported answers for a team of 2 with a reason when the driver
    refuses (this single-GPU box: cuMulticastCreate rejects every team size,
    profiles/r02_probe_mc2.txt); with >= 2 GPUs the NVLS parity test in
    test_gpu_multiproc.py runs instead of skipping."""
    F = _F()
    ok, gran, why = F.mc_supported(2, 64 << 20)
    assert ok or why
    if ok:
        assert gran > 0 and gran % (2 << 20) == 0


def test_single_bucket_gpu_after_mixed_gpu():
    """Regression (found by tests/test_gpu_fuzz.py, seed 82): with the mixed
    work order, a GPU whose atoms go to several destination groups leaves
    holes in the mixed slot space, so a later GPU whose atoms all go to one
    group starts at different offsets in the two spaces; launched alone (one
    process per GPU: kv_reshard(plan, g)) it must still map its slots.  The
    fuzz case itself (16-byte atoms, 16 pools), plus the multi-process
    'hetero' cases in test_gpu_multiproc.py."""
    geo = (2, 16, 16, 1, 1)
    spec = [(166, (1, 1), (14, 1)),
            (3, (0, 16), (0, 4), [0, 14, 4, 15, 1, 2, 6, 8, 3, 11, 10, 13, 5, 12, 7, 9], None),
            (1, (4, 4), (0, 16), [0, 3, 1, 2], None),
            (0, (0, 16), (0, 16)),
            (233, (15, 1), (0, 16))]
    run_parity(geo, [870] * 16, spec, seed=82, per_gpu_launch=True, work_order=1)
