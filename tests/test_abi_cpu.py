"""C-ABI library on CPU (no GPU needed): it loads, exports every symbol
include/flykv.h declares, and its host logic (validation, allocator, planner,
byte matrix, weight views) matches the oracle and the paper's rules.
No compute call is made here (pool pointers are fake, never dereferenced)."""
import os
import re

import numpy as np
import pytest

from helpers import oracle_alloc
from oracle import oracle as O
from paper_2602_22593_b200 import flykv as F

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_symbols_exported():
    hdr = open(os.path.join(ROOT, "include", "flykv.h")).read()
    names = set(re.findall(r"^\s*(?:kv_status|void|const char\*|int64_t)\s+\**(\w+)\s*\(", hdr, re.M))
    assert {"kv_plan_switch", "kv_reshard", "kv_remap_block_tables", "weight_shard_view"} <= names
    for n in names:
        assert hasattr(F._lib, n), n
    assert set(F.EXPORTED) == names


def fake_cache(geo, nb, degrees=(2, 4, 8)):
    g = F.geometry(*geo)
    bases = [[(1 << 40) + (gpu << 36) + (l << 30) for l in range(geo[0])] for gpu in range(len(nb))]
    return F.KVCache(g, nb, bases, degrees)


def test_layout_matches_oracle():
    for H in (1, 2, 4, 8):
        for p in (1, 2, 4, 8, 16):
            g = F.geometry(3, H, 64, 16, 2)
            og = O.Geom(3, H, 64, 16, 2)
            hl, bt, M = F.kv_layout(g, p)
            assert (hl, bt, M) == (O.h_loc(og, p), O.block_tokens(og, p), O.block_bytes(og))
            for T in (0, 1, 16, 17, 1000):
                assert F.kv_blocks_for(g, T, p) == O.num_blocks(og, T, p)
    with pytest.raises(F.FlyKVError) as e:
        F.kv_layout(F.geometry(1, 8, 64, 16, 2), 3)
    assert e.value.name == "KV_ERR_INDIVISIBLE_DEGREE"


def test_alloc_lowest_uniform_and_conservation():
    c = fake_cache((2, 4, 8, 4, 2), [16, 16])
    a = c.alloc((0, 1), 3)
    assert list(a) == [0, 1, 2]
    b = c.alloc((1, 1), 2)
    assert list(b) == [0, 1]
    t = c.alloc((0, 2), 3)          # lowest free on both GPUs (R6, R8)
    assert list(t) == [3, 4, 5]
    c.free((0, 1), [1])
    t2 = c.alloc((0, 2), 2)         # 1 is free on GPU0 but held on GPU1
    assert list(t2) == [6, 7]
    assert c.free_count(0) == 16 - 7 and c.free_count(1) == 16 - 7
    with pytest.raises(F.FlyKVError) as e:
        c.alloc((0, 2), 100)
    assert e.value.name == "KV_ERR_OUT_OF_BLOCKS"
    with pytest.raises(F.FlyKVError):
        c.free((0, 1), [1])         # not held any more
    with pytest.raises(F.FlyKVError) as e:
        c.alloc((1, 2), 1)          # unaligned group
    assert e.value.name == "KV_ERR_UNKNOWN_GROUP"


def _random_case(rng, H, n_gpus, n_req, degrees, nb):
    T = rng.integers(0, 90, size=n_req)
    spec = []
    for i in range(n_req):
        p0 = int(rng.choice(degrees))
        p1 = int(rng.choice(degrees))
        g0 = int(rng.integers(0, n_gpus // p0)) * p0
        g1 = int(rng.integers(0, n_gpus // p1)) * p1
        spec.append((int(T[i]), (g0, p0), (g1, p1)))
    return spec


@pytest.mark.parametrize("seed", range(12))
def test_plan_tables_match_oracle(seed):
    """The product's host allocator/planner chooses exactly the oracle's
    destination tables (R6, R8) and leaves the same held sets (R13)."""
    rng = np.random.default_rng(seed)
    H = [1, 2, 4, 8][seed % 4]
    n_gpus = 8
    geo = (2, H, 4, 4, 2)
    og = O.Geom(*geo)
    nb = [256] * n_gpus
    spec = _random_case(rng, H, n_gpus, 10, [1, 2, 4, 8], nb)
    c = fake_cache(geo, nb)
    M = O.block_bytes(og)
    pools = [np.zeros(geo[0] * n * M, dtype=np.uint8) for n in nb]
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    oreqs, freqs = [], []
    for i, (T, src, dst) in enumerate(spec):
        n = O.num_blocks(og, T, src[1])
        ids = oracle_alloc(c, held, src, n)   # oracle-chosen IDs, checked against kv_alloc
        oreqs.append(O.Req(T, src, list(ids), dst))
        freqs.append((100 + i, T, src, ids, dst))
    for g in range(n_gpus):
        assert np.array_equal(c.held_mask(g), held[g])
    st, otabs = O.switch(og, pools, held, oreqs)
    if st != 0:  # both sides must refuse, and the product must change nothing
        before = [c.held_mask(g).copy() for g in range(n_gpus)]
        with pytest.raises(F.FlyKVError) as e:
            c.plan_switch(freqs)
        assert e.value.name == "KV_ERR_OUT_OF_BLOCKS"
        assert all(np.array_equal(c.held_mask(g), before[g]) for g in range(n_gpus))
        return
    plan = c.plan_switch(freqs)
    ftabs = plan.dst_tables()
    assert [list(a) for a in ftabs] == [list(b) for b in otabs]
    # residency sizes agree with the oracle's CSR tables
    for g in range(n_gpus):
        rp, ids, meta = O.tables(og, g, oreqs, otabs)
        assert plan.resident(g) == (len(meta), len(ids))
    # a plan that is never committed rolls back on destroy
    plan.destroy()
    for g in range(n_gpus):
        hm = c.held_mask(g)
        want = np.zeros(nb[g], dtype=np.uint8)
        for (T, src, ids_, dst) in [(f[1], f[2], f[3], f[4]) for f in freqs]:
            if src[0] <= g < src[0] + src[1]:
                want[ids_] = 1
        assert np.array_equal(hm, want)


def test_plan_validation_errors():
    geo = (2, 4, 8, 4, 2)
    c = fake_cache(geo, [32, 32, 32, 32])
    a = c.alloc((0, 1), 3)   # T up to 12
    b = c.alloc((1, 1), 2)
    def expect(reqs, name):
        before = [c.held_mask(g).copy() for g in range(4)]
        with pytest.raises(F.FlyKVError) as e:
            c.plan_switch(reqs)
        assert e.value.name == name, e.value
        for g in range(4):
            assert np.array_equal(c.held_mask(g), before[g])

    expect([(1, 12, (0, 1), a[:2], (0, 2))], "KV_ERR_BAD_BLOCK_TABLE")        # wrong length
    expect([(1, 12, (0, 1), [a[0], a[1], 31], (0, 2))], "KV_ERR_BAD_BLOCK_TABLE")  # 31 not held
    expect([(1, 12, (0, 1), [a[0], a[1], 99], (0, 2))], "KV_ERR_BAD_BLOCK_TABLE")  # out of range
    expect([(1, 12, (0, 1), a, (1, 2))], "KV_ERR_UNKNOWN_GROUP")              # unaligned
    expect([(1, 12, (0, 1), a, (0, 3))], "KV_ERR_UNKNOWN_GROUP")              # degree not in P
    expect([(1, 12, (0, 1), a, (0, 2)), (1, 8, (1, 1), b, (0, 2))], "KV_ERR_DUPLICATE_REQUEST")
    expect([(1, 12, (0, 1), a, (0, 2)), (2, 12, (0, 1), a, (0, 2))], "KV_ERR_BAD_BLOCK_TABLE")  # shared (R14)
    expect([(1, -1, (0, 1), [], (0, 2))], "KV_ERR_INVALID_ARG")
    # out of blocks is transactional: first request fits, second does not
    big = c.alloc((2, 1), 30)
    expect([(1, 12, (0, 1), a, (0, 2)), (2, 120, (2, 1), big, (2, 2))], "KV_ERR_OUT_OF_BLOCKS")


def test_gqa_degree_rules():
    c = fake_cache((1, 2, 8, 4, 2), [16] * 8, degrees=(2, 4, 8))
    a = c.alloc((0, 1), 2)
    plan = c.plan_switch([(1, 8, (0, 1), a, (0, 8))])   # 8 > H=2 -> replication x4
    st, mat = plan.stats()
    # B(8) = H*B = 8 -> one block per rank; every rank receives one head copy
    assert [len(t) for t in plan.dst_tables()] == [1]
    assert st["n_atoms"] == 1 * 2 * 2 * 2            # L*2*C*H
    assert st["n_atom_writes"] == st["n_atoms"] * 4
    assert (mat[0] > 0).sum() == 8
    plan.destroy()
    with pytest.raises(F.FlyKVError) as e:
        fake_cache((1, 3, 8, 4, 2), [4] * 2, degrees=(2,))
    assert e.value.name == "KV_ERR_INDIVISIBLE_DEGREE"


def test_byte_matrix_matches_atom_enumeration():
    """kv_plan_get_stats byte matrix == counting every atom with the oracle's owner map."""
    rng = np.random.default_rng(3)
    geo = (3, 4, 8, 4, 2)
    og = O.Geom(*geo)
    n_gpus = 8
    c = fake_cache(geo, [128] * n_gpus)
    spec = _random_case(rng, 4, n_gpus, 12, [1, 2, 4, 8], None)
    reqs = []
    mirror = [np.zeros(128, dtype=np.uint8) for _ in range(n_gpus)]
    for i, (T, src, dst) in enumerate(spec):
        ids = oracle_alloc(c, mirror, src, O.num_blocks(og, T, src[1]))
        reqs.append((i, T, src, ids, dst))
    plan = c.plan_switch(reqs)
    st, mat = plan.stats()
    want = np.zeros((n_gpus, n_gpus), dtype=np.int64)
    atom = og.B * og.d * og.e
    tabs = plan.dst_tables()
    for (i, T, src, ids, dst), t1 in zip(reqs, tabs):
        if src == dst:
            continue
        for h in range(og.H):
            sg = src[0] + O.owner_rank(og, src[1], h, 0)
            for j in range(O.replicas(og, dst[1])):
                dg = dst[0] + O.owner_rank(og, dst[1], h, j)
                want[sg, dg] += og.L * 2 * (-(-T // og.B)) * atom
    assert np.array_equal(mat, want)
    assert st["payload_bytes"] == want.sum()
    plan.destroy()


def test_weight_views_match_oracle():
    from oracle import weights as W
    Hq, Hkv, d, hidden = 8, 2, 4, 16
    rows = (Hq + 2 * Hkv) * d
    base = 1 << 32
    full = np.arange(rows * hidden).reshape(rows, hidden)
    for m in (1, 2, 4, 8):
        for r in range(m):
            v = F.weight_shard_view(F.weight_desc(base, rows, hidden, 2, F.KV_W_QKV, num_q_heads=Hq,
                                                  num_kv_heads=Hkv, head_dim=d), r, m)
            ref = W.view_qkv(full, r, m, Hq, Hkv, d)
            assert v.n_seg == 3
            for s, rs in zip(v.segments(), ref):
                # the segment addresses exactly the oracle's rows (zero-copy alias)
                r0 = (s.ptr - base) // (2 * hidden)
                assert np.array_equal(full[r0:r0 + s.rows, :s.cols], rs)
                assert s.row0 == r0 and s.ld == hidden
    Wf = np.arange(6 * 8).reshape(6, 8)
    for m in (1, 2, 4, 8):
        for r in range(m):
            v = F.weight_shard_view(F.weight_desc(base, 6, 8, 4, F.KV_W_ROW), r, m)
            (ref,) = W.view_row(Wf, r, m)
            s = v.seg[0]
            c0 = (s.ptr - base) // 4
            assert s.col0 == c0 and np.array_equal(Wf[:, c0:c0 + s.cols], ref) and s.ld == 8
            v = F.weight_shard_view(F.weight_desc(base, 8, 6, 4, F.KV_W_COLUMN), r, m)
            (ref,) = W.view_col(np.arange(48).reshape(8, 6), r, m)
            assert v.seg[0].rows == ref.shape[0] and v.seg[0].row0 == r * 8 // m
    with pytest.raises(F.FlyKVError) as e:
        F.weight_shard_view(F.weight_desc(base, 6, 8, 4, F.KV_W_ROW), 0, 3)
    assert e.value.name == "KV_ERR_INDIVISIBLE_EXTENT"
    with pytest.raises(F.FlyKVError) as e:
        F.weight_shard_view(F.weight_desc(base, 6, 8, 4, F.KV_W_ROW), 4, 4)
    assert e.value.name == "KV_ERR_RANK_OUT_OF_RANGE"


def test_memory_bounded_waves_match_oracle():
    """a DP -> TP8 promotion that does not fit in one shot
    (OUT_OF_BLOCKS) succeeds in waves; every wave's tables equal the oracle's
    allocator applied wave after wave, and allocator states agree."""
    geo = (2, 8, 8, 4, 2)
    og = O.Geom(*geo)
    n_gpus, nb = 8, [56] * 8
    c = fake_cache(geo, nb)
    rng = np.random.default_rng(9)
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    reqs = []
    for i in range(24):
        T = int(rng.integers(20, 50))
        src = (i % n_gpus, 1)
        ids = oracle_alloc(c, held, src, O.num_blocks(og, T, 1))
        reqs.append((i, T, src, ids, (0, 8)))
    with pytest.raises(F.FlyKVError) as e:
        c.plan_switch(reqs)
    assert e.value.name == "KV_ERR_OUT_OF_BLOCKS"
    waves = F.kv_plan_waves(c, reqs)
    assert len(waves) > 1 and waves[0][0] == 0 and waves[-1][1] == len(reqs)
    assert all(a < b for a, b in waves) and all(waves[k][1] == waves[k + 1][0] for k in range(len(waves) - 1))
    for a, b in waves:
        plan = c.plan_switch(reqs[a:b])
        st, otabs = O.switch(og, None, held, [O.Req(T, s, list(ids), d) for (_, T, s, ids, d) in reqs[a:b]],
                             copy=False)
        assert st == 0
        assert [list(x) for x in plan.dst_tables()] == [list(y) for y in otabs]
        plan.commit()
        for g in range(n_gpus):
            assert np.array_equal(c.held_mask(g), held[g])
    # a byte cap splits further
    c2 = fake_cache(geo, [4096] * 8)
    reqs2 = []
    for i in range(8):
        ids = c2.alloc((i, 1), F.kv_blocks_for(c2.geom, 64, 1))
        reqs2.append((i, 64, (i, 1), ids, (0, 8)))
    one = 2 * 2 * 8 * 64 * 8 * 2   # L*2*H*T*d*e per request
    assert len(F.kv_plan_waves(c2, reqs2)) == 1
    assert [b - a for a, b in F.kv_plan_waves(c2, reqs2, max_wave_bytes=3 * one)] == [3, 3, 2]


def test_rank_ids_plan_and_suggestion():
    """N2: the product's planner follows per-request rank IDs exactly like the
    oracle (destination tables, byte matrix); kv_suggest_rank_ids finds the
    assignment that keeps half of a TP4 -> TP8 promotion local (vs 1/8)."""
    geo = (2, 8, 8, 4, 2)
    og = O.Geom(*geo)
    c = fake_cache(geo, [256] * 8)
    reqs = []
    mirror = [np.zeros(256, dtype=np.uint8) for _ in range(8)]
    for i, T in enumerate([64, 130, 7]):
        ids = oracle_alloc(c, mirror, (0, 4), O.num_blocks(og, T, 4))
        reqs.append((i, T, (0, 4), ids, (0, 8)))
    sugg = F.kv_suggest_rank_ids(c, reqs, (0, 8))
    assert sorted(sugg) == list(range(8))
    assert all(sugg[m] // 2 == m for m in range(4))   # member m < 4 owns one of its own two heads
    for rid, local in ((None, 1 / 8), (sugg, 1 / 2)):
        rq = [r + (None, rid) for r in reqs]
        plan = c.plan_switch(rq)
        st, mat = plan.stats()
        assert np.trace(mat) / mat.sum() == pytest.approx(local)
        # byte matrix equals the oracle's atom map
        want = np.zeros((8, 8), dtype=np.int64)
        tabs = plan.dst_tables()
        for (i, T, s_, ids, d_), t in zip(reqs, tabs):
            sg, so, dg, do = O.atom_map(og, [256] * 8, T, s_, ids, d_, t, None, rid)
            np.add.at(want, (sg, dg), og.B * og.d * og.e)
        assert np.array_equal(mat, want)
        plan.destroy()
    with pytest.raises(F.FlyKVError) as e:
        c.plan_switch([reqs[0] + (None, [0, 1, 2, 3, 4, 5, 6, 6])])
    assert e.value.name == "KV_ERR_INVALID_ARG"


def test_plan_state_machine():
    """kv_plan_commit releases sources once (idempotent); a committed plan
    refuses kv_reshard (its sources may be reused, BAD_STATE) and destroy
    keeps the destination allocation."""
    c = fake_cache((1, 4, 8, 4, 2), [32, 32])
    a = c.alloc((0, 1), 3)
    plan = c.plan_switch([(1, 12, (0, 1), a, (0, 2))])
    held_planned = [c.held_mask(g).sum() for g in (0, 1)]
    plan.commit()
    plan.commit()
    assert [c.held_mask(g).sum() for g in (0, 1)] == [held_planned[0] - 3, held_planned[1]]
    with pytest.raises(F.FlyKVError) as e:
        F.kv_reshard(plan, -1)
    assert e.value.name == "KV_ERR_BAD_STATE"
    dst = plan.dst_tables()[0]
    plan.destroy()
    assert all(c.held_mask(g)[dst].all() for g in (0, 1))


def test_pack_unpack_argument_errors():
    """kv_pack / kv_unpack validate before touching the device: NULL buffer
    or offsets -> INVALID_ARG, GPU out of range -> INVALID_ARG, committed plan
    -> BAD_STATE; a2a_offsets gives the all_to_all_single prefixes."""
    c = fake_cache((1, 4, 8, 4, 2), [32, 32])
    a = c.alloc((0, 1), 3)
    plan = c.plan_switch([(1, 12, (0, 1), a, (0, 2))])
    for fn in (F.kv_pack, F.kv_unpack):
        with pytest.raises(F.FlyKVError) as e:
            fn(plan, 0, 0, [0, 0])
        assert e.value.name == "KV_ERR_INVALID_ARG"
        with pytest.raises(F.FlyKVError) as e:
            fn(plan, 2, 1 << 40, [0, 0])
        assert e.value.name == "KV_ERR_INVALID_ARG"
    _, mat = plan.stats()
    send, recv = F.a2a_offsets(plan)
    # chunk (s -> d) sits at send[s][d] in s's send buffer and at recv[d][s] in d's receive buffer
    assert send[0][0] == 0 and send[0][1] == mat[0][0] and recv[1][0] == 0 and recv[1][1] == mat[0][1]
    plan.commit()
    for fn in (F.kv_pack, F.kv_unpack):
        with pytest.raises(F.FlyKVError) as e:
            fn(plan, 0, 1 << 40, [0, 0])
        assert e.value.name == "KV_ERR_BAD_STATE"


def test_free_ten_thousand_random_requests():
    """SPEC S:236 / S:250: 10,000 random requests admitted into random aligned
    groups and freed in random order; allocated + free == num_blocks on every
    GPU after every operation, the product's choices equal the oracle's
    allocator, and the pools end empty."""
    from oracle import brute
    nb = 400
    c = fake_cache((1, 8, 8, 4, 2), [nb] * 8)
    og = O.Geom(1, 8, 8, 4, 2)
    held = [np.zeros(nb, dtype=np.uint8) for _ in range(8)]
    rng = np.random.default_rng(236)
    live = []
    admitted = 0
    while admitted < 10000:
        if live and (rng.random() < 0.45 or len(live) > 60):
            grp, ids = live.pop(int(rng.integers(len(live))))
            c.free(grp, ids)
            for r in range(grp[1]):
                held[grp[0] + r][ids] = 0
        else:
            p = int(rng.choice([1, 2, 4, 8]))
            grp = (int(rng.integers(8 // p)) * p, p)
            n = O.num_blocks(og, int(rng.integers(1, 200)), p)
            want = brute.lowest_common_free(held, grp, n)
            if want is None:
                continue
            ids = c.alloc(grp, n)
            assert list(ids) == list(want)
            for r in range(p):
                held[grp[0] + r][ids] = 1
            live.append((grp, ids))
            admitted += 1
        for g in range(8):
            assert c.free_count(g) + int(held[g].sum()) == nb
    for grp, ids in live:
        c.free(grp, ids)
    assert all(c.free_count(g) == nb for g in range(8))


def test_kv_switch_errors_before_the_device():
    """kv_switch fails in planning with no state change (OUT_OF_BLOCKS), and
    kv_switch_back refuses an uncommitted plan (BAD_STATE) or a plan of
    another cache (INVALID_ARG) -- all before any device work."""
    c = fake_cache((1, 4, 8, 4, 2), [8, 8])
    a = c.alloc((0, 1), 6)
    before = [c.held_mask(g).copy() for g in (0, 1)]
    with pytest.raises(F.FlyKVError) as e:
        F.kv_switch(c, [(1, 24, (0, 1), a, (0, 2))])   # needs 3 blocks on both GPUs; GPU 0 has 2 free
    assert e.value.name == "KV_ERR_OUT_OF_BLOCKS"
    assert all(np.array_equal(c.held_mask(g), before[g]) for g in (0, 1))
    plan = c.plan_switch([(1, 8, (0, 1), a[:2], (0, 2))])
    with pytest.raises(F.FlyKVError) as e:
        F.kv_switch_back(c, plan)
    assert e.value.name == "KV_ERR_BAD_STATE"
    other = fake_cache((1, 4, 8, 4, 2), [8, 8])
    plan.commit()
    with pytest.raises(F.FlyKVError) as e:
        F.kv_switch_back(other, plan)
    assert e.value.name == "KV_ERR_INVALID_ARG"
    with pytest.raises(F.FlyKVError) as e:
        plan.host_tables(0)   # not run by kv_switch
    assert e.value.name == "KV_ERR_BAD_STATE"


def test_kv_switch_multi_errors_before_the_device():
    """kv_switch_multi: no waves is a no-op; a wave that does not fit fails in
    its planning with no state change and no plan returned -- before any
    device work."""
    c = fake_cache((1, 4, 8, 4, 2), [8, 8])
    assert F.kv_switch_multi(c, []) == []
    a = c.alloc((0, 1), 6)
    before = [c.held_mask(g).copy() for g in (0, 1)]
    with pytest.raises(F.FlyKVError) as e:
        F.kv_switch_multi(c, [[(1, 24, (0, 1), a, (0, 2))]])
    assert e.value.name == "KV_ERR_OUT_OF_BLOCKS"
    assert all(np.array_equal(c.held_mask(g), before[g]) for g in (0, 1))


def _run_pieces_against_oracle(c, og, held, reqs, waves, n_gpus):
    """Execute kv_plan_pieces' waves on the product (plan + commit per wave,
    fake pointers) and on the oracle's allocator with the same piece
    requests; tables and allocator state must agree wave by wave.  Returns
    each request's concatenated destination table."""
    parts = [[] for _ in reqs]
    for wave in waves:
        sub = [F.piece_request(c.geom, reqs[i], t0, t1) for i, t0, t1 in wave]
        plan = c.plan_switch(sub)
        st, otabs = O.switch(og, None, held, [O.Req(T, s, list(ids), d) for (_, T, s, ids, d) in sub], copy=False)
        assert st == 0
        assert [list(x) for x in plan.dst_tables()] == [list(y) for y in otabs]
        plan.commit()
        for g in range(n_gpus):
            assert np.array_equal(c.held_mask(g), held[g])
        for (i, _, _), t in zip(wave, otabs):
            parts[i].append(np.asarray(t, dtype=np.int32))
    return [np.concatenate(p) for p in parts]


def test_pieces_equal_waves_when_requests_fit():
    """kv_plan_pieces keeps requests whole, in kv_plan_waves' partition, when
    every request fits a fresh wave (R20 reduces to N1)."""
    geo = (2, 8, 8, 4, 2)
    og = O.Geom(*geo)
    nb = [56] * 8
    c = fake_cache(geo, nb)
    rng = np.random.default_rng(9)
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    reqs = []
    for i in range(24):
        T = int(rng.integers(20, 50))
        ids = oracle_alloc(c, held, (i % 8, 1), O.num_blocks(og, T, 1))
        reqs.append((i, T, (i % 8, 1), ids, (0, 8)))
    waves = F.kv_plan_waves(c, reqs)
    pieces = F.kv_plan_pieces(c, reqs)
    assert [[(i, 0, reqs[i][1]) for i in range(a, b)] for a, b in waves] == pieces


def test_one_long_request_promoted_in_pieces():
    """R20 / Use Case 3: one long TP4 request that fills most of
    GPUs 0-3 is promoted to TP8.  Its source and destination cannot coexist
    (one shot and request-granular waves both fail with OUT_OF_BLOCKS), but
    block-aligned token pieces over several waves succeed: the pieces tile
    [0, T) on whole blocks of both layouts, every wave's allocation equals
    the oracle's, and the concatenated table has ceil(T / B(8)) blocks."""
    geo = (2, 8, 8, 4, 2)
    og = O.Geom(*geo)
    nb = [80] * 8
    c = fake_cache(geo, nb)
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    T = 66 * 16 + 5                       # B(4) = 16 tokens: 67 blocks on each of GPUs 0-3
    ids = oracle_alloc(c, held, (0, 4), O.num_blocks(og, T, 4))
    reqs = [(0, T, (0, 4), ids, (0, 8))]
    with pytest.raises(F.FlyKVError) as e:
        c.plan_switch(reqs)
    assert e.value.name == "KV_ERR_OUT_OF_BLOCKS"
    with pytest.raises(F.FlyKVError):
        F.kv_plan_waves(c, reqs)
    waves = F.kv_plan_pieces(c, reqs)
    assert len(waves) >= 2 and all(len(w) == 1 for w in waves)
    bounds = [w[0][1:] for w in waves]
    assert bounds[0][0] == 0 and bounds[-1][1] == T
    assert all(bounds[k][1] == bounds[k + 1][0] for k in range(len(bounds) - 1))
    unit = 4 * 8                          # whole blocks of both layouts: B(8) = 32 tokens
    assert all(t1 % unit == 0 for _, t1 in bounds[:-1])
    final = _run_pieces_against_oracle(c, og, held, reqs, waves, 8)
    assert len(final[0]) == O.num_blocks(og, T, 8)
    assert all(c.free_count(g) + int(held[g].sum()) == nb[g] for g in range(8))
    # a byte bound splits a request that would fit into more waves
    c2 = fake_cache(geo, [4096] * 8)
    held2 = [np.zeros(4096, dtype=np.uint8) for _ in range(8)]
    ids2 = oracle_alloc(c2, held2, (0, 1), O.num_blocks(og, 1000, 1))
    per_token = 2 * 2 * 8 * 8 * 2                      # L * 2 * H * d * e
    w2 = F.kv_plan_pieces(c2, [(0, 1000, (0, 1), ids2, (0, 8))], max_wave_bytes=300 * per_token)
    assert len(w2) >= 4 and all((t1 - t0) * per_token <= 300 * per_token for [(_, t0, t1)] in w2)
    _run_pieces_against_oracle(c2, og, held2, [(0, 1000, (0, 1), ids2, (0, 8))], w2, 8)


def test_kv_switch_waves_schedule_retry_before_the_device():
    """kv_switch_waves grows its piece buffer when the schedule needs more
    pieces than the first guess (a byte cap of 1 cuts every request into
    block-aligned pieces, many more than 2 x requests), then plans the first
    wave.  On a CPU-only host the device step then fails with KV_ERR_CUDA and
    the failed wave's allocations are rolled back: no state change."""
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("checks the no-device failure path")
    c = fake_cache((1, 4, 8, 4, 2), [256, 256])
    a = c.alloc((0, 1), 40)              # 160 tokens at B = 4
    before = [c.held_mask(g).copy() for g in (0, 1)]
    reqs = [(1, 160, (0, 1), a, (0, 2))]
    assert sum(len(w) for w in F.kv_plan_pieces(c, reqs, 1)) > 16   # beyond the binding's first buffer
    with pytest.raises(F.FlyKVError) as e:
        F.kv_switch_waves(c, reqs, max_wave_bytes=1, split=True)
    assert e.value.name == "KV_ERR_CUDA"
    assert all(np.array_equal(c.held_mask(g), before[g]) for g in (0, 1))


def test_empty_wave_schedules():
    """An empty request list has no waves: kv_plan_waves writes only
    wave_start[0] (it used to write one entry past n_reqs + 1),
    and kv_switch_waves(split=False) of nothing is a no-op that needs no
    device."""
    c = fake_cache((1, 4, 8, 4, 2), [64, 64])
    assert F.kv_plan_waves(c, []) == []
    waves, plans = F.kv_switch_waves(c, [], split=False)
    assert waves == [] and plans == []
    assert F.kv_plan_pieces(c, []) == []


def test_cache_close_detaches_live_plans():
    """KVCache.close() while a plan is alive detaches the plan:
    calls on it return BAD_STATE instead of touching freed allocator state,
    and destroying it afterwards is safe."""
    c = fake_cache((1, 4, 8, 4, 2), [64, 64])
    a = c.alloc((0, 1), 5)
    plan = c.plan_switch([(1, 20, (0, 1), a, (0, 2))])
    assert plan.resident(0) == (1, 3)
    c.close()
    with pytest.raises(F.FlyKVError) as e:
        plan.resident(0)
    assert e.value.name == "KV_ERR_BAD_STATE"
    with pytest.raises(F.FlyKVError):
        plan.commit()
    assert len(plan.dst_tables()[0]) == 3         # host-side plan data stays readable
    plan.destroy()
    plan.destroy()


def test_a2a_offsets_are_exclusive_prefixes():
    """kv_plan_a2a_offsets on a 4-GPU merge + split plan: send_off rows,
    recv_off columns and the packed row-major layout are the exclusive
    prefix sums of the plan's bytes matrix (written out here with numpy)."""
    c = fake_cache((2, 8, 16, 4, 2), [64] * 4)
    reqs = []
    for i, (src, dst) in enumerate([((0, 1), (0, 4)), ((1, 1), (2, 2)), ((2, 2), (0, 1)), ((3, 1), (0, 2))]):
        T = 9 + 7 * i
        reqs.append((i, T, src, c.alloc(src, F.kv_blocks_for(c.geom, T, src[1])), dst))
    plan = c.plan_switch(reqs)
    _, m = plan.stats()
    send, recv, packed = plan.a2a_offsets()
    n = m.shape[0]
    for s_ in range(n):
        for d in range(n):
            assert send[s_, d] == m[s_, :d].sum()
            assert recv[d, s_] == m[:s_, d].sum()
            assert packed[s_, d] == m.reshape(-1)[:s_ * n + d].sum()


def test_piece_request_slices_the_source_table():
    """kv_piece_request: tokens [tok0, tok1) of a request start at source
    block tok0 / B(p0) (Eq.2: B(2) = 2B here) and span ceil(tok1 / B(p0)) -
    tok0 / B(p0) blocks; the whole range is the request itself; a piece that
    does not start on a source block is rejected."""
    g = F.geometry(1, 4, 8, 4, 2)
    ids = np.arange(100, 113, dtype=np.int32)          # 13 blocks of B(2) = 8 tokens: 100 tokens
    req = (7, 100, (0, 2), ids, (0, 4))
    p = F.piece_request(g, req, 16, 50)
    assert p[0] == 7 and p[1] == 34 and p[2] == (0, 2) and p[4] == (0, 4)
    assert list(p[3]) == list(range(102, 107))          # blocks 2 .. ceil(50/8)-1 = 6
    whole = F.piece_request(g, req, 0, 100)
    assert whole[:3] == req[:3] and list(whole[3]) == list(ids) and whole[4] == req[4]
    with pytest.raises(F.FlyKVError):
        F.piece_request(g, req, 12, 50)
    with pytest.raises(F.FlyKVError):
        F.piece_request(g, req, 16, 101)


def test_packed_offsets_are_the_documented_prefixes():
    """kv_plan_packed_offsets: pool g's slice of the packed remap outputs
    starts at req_ptr sum_{g'<g}(n_res[g'] + 1), block_ids sum n_ids[g'],
    meta 4 * sum n_res[g'] (include/flykv.h, kv_remap_block_tables)."""
    c = fake_cache((2, 8, 16, 4, 2), [64] * 4)
    reqs = []
    for i, (src, dst) in enumerate([((0, 1), (0, 4)), ((1, 1), (2, 2)), ((2, 2), (0, 1)), ((3, 1), (0, 2))]):
        T = 11 + 9 * i
        reqs.append((i, T, src, c.alloc(src, F.kv_blocks_for(c.geom, T, src[1])), dst))
    plan = c.plan_switch(reqs)
    off, tot = plan.packed_offsets()
    res = [plan.resident(g) for g in range(4)]
    for g in range(4):
        assert off[g, 0] == sum(r + 1 for r, _ in res[:g])
        assert off[g, 1] == sum(i for _, i in res[:g])
        assert off[g, 2] == 4 * sum(r for r, _ in res[:g])
    assert list(tot) == [sum(r for r, _ in res) + 4, sum(i for _, i in res), 4 * sum(r for r, _ in res)]


def test_round2_entry_points_validate_before_the_device():
    """Argument checks of this round's entry points need no GPU: bad pool
    ranges (kv_reshard_range, kv_switch_range, kv_switch_range_host), barrier
    arguments (kv_group_barrier, kv_group_barrier_selftest), multicast teams (kv_cache_set_multicast), strict-mode
    flags; kv_verify_replicas of a plan without replicated sources is (0,
    none) without touching the device."""
    c = fake_cache((1, 4, 8, 4, 2), [64] * 4)
    a = c.alloc((0, 1), 5)
    reqs = [(1, 20, (0, 1), a, (0, 2))]
    plan = c.plan_switch(reqs)
    for lo, hi in ((0, 0), (-1, 2), (2, 5), (3, 1)):
        with pytest.raises(F.FlyKVError) as e:
            F.kv_reshard_range(plan, lo, hi)
        assert e.value.name == "KV_ERR_INVALID_ARG"
    assert F.kv_verify_replicas(plan) == (0, None)
    plan.destroy()
    with pytest.raises(F.FlyKVError) as e:
        F.kv_switch_range(c, reqs, 2, 9)
    assert e.value.name == "KV_ERR_INVALID_ARG"
    called = []   # kv_switch_range_host: the same checks, the callback never runs
    with pytest.raises(F.FlyKVError) as e:
        F.kv_switch_range(c, reqs, 2, 9, lambda: called.append(1))
    assert e.value.name == "KV_ERR_INVALID_ARG" and not called
    for n, rounds, absent, tmo in ((0, 1, -1, 1), (65, 1, -1, 1), (2, 0, -1, 1), (2, 1, 2, 1), (2, 1, -1, 0)):
        with pytest.raises(F.FlyKVError) as e:   # barrier self-test arguments, before any device work
            F.group_barrier_selftest(n, rounds, absent, tmo)
        assert e.value.name == "KV_ERR_INVALID_ARG"
    assert all(c.free_count(g) == 64 - (5 if g == 0 else 0) for g in range(4))   # nothing planned
    for args in (([], 0, 1), ([1 << 40], 1, 1), ([1 << 40 | 4], 0, 1), ([1 << 40], 0, 0)):
        flags, me, tmo = args
        with pytest.raises(F.FlyKVError) as e:
            F.kv_group_barrier(flags, me, 1, tmo)
        assert e.value.name == "KV_ERR_INVALID_ARG"
    bases = [1 << 40]
    for team, mode in (((1, 2), 1), ((0, 1), 1), ((0, 8), 1), ((0, 2), 3)):
        with pytest.raises(F.FlyKVError):
            c.set_multicast(team, bases, mode)
    c.set_multicast((2, 2), bases, 2)
    with pytest.raises(F.FlyKVError):
        c.set_multicast((0, 2), bases, 1)          # one mode per cache
    c.set_multicast((2, 2), None, 2)               # cleared: the mode is free again
    c.set_multicast((0, 2), bases, 1)
    assert F._lib.kv_cache_set_strict(c._h, 2) == 1          # KV_ERR_INVALID_ARG: strict is 0 or 1
    c.set_strict(True)
    c.set_strict(False)


def test_weight_views_fuzz_against_oracle():
    """Random fused-QKV, column- and row-parallel shapes (incl. GQA m > H_kv,
    padded leading dimensions, 1/2/4-byte elements): every segment of
    weight_shard_view addresses exactly the rows / columns of the numpy
    oracle's Eq.1 view, or both reject the same way."""
    from oracle import weights as W
    rng = np.random.default_rng(2024)
    base = 1 << 36
    for _ in range(400):
        e = int(rng.choice([1, 2, 4]))
        m = int(rng.choice([1, 2, 4, 8, 16]))
        r = int(rng.integers(0, m))
        kind = int(rng.integers(0, 3))
        if kind == F.KV_W_QKV:
            Hkv = int(rng.choice([1, 2, 4, 8]))
            Hq = Hkv * int(rng.choice([1, 2, 4, 8]))
            d = int(rng.choice([1, 2, 4]))
            hidden = int(rng.integers(1, 9))
            rows = (Hq + 2 * Hkv) * d
            ld = hidden + int(rng.integers(0, 3))
            full = np.arange(rows * ld).reshape(rows, ld)
            try:
                ref = W.view_qkv(full[:, :hidden], r, m, Hq, Hkv, d)
            except (W.RankOutOfRange, W.IndivisibleExtent) as ex:
                with pytest.raises(F.FlyKVError):
                    F.weight_shard_view(F.weight_desc(base, rows, hidden, e, kind, ld=ld, num_q_heads=Hq,
                                                      num_kv_heads=Hkv, head_dim=d), r, m)
                continue
            v = F.weight_shard_view(F.weight_desc(base, rows, hidden, e, kind, ld=ld, num_q_heads=Hq,
                                                  num_kv_heads=Hkv, head_dim=d), r, m)
            assert v.n_seg == len(ref)
            for s, rs in zip(v.segments(), ref):
                r0 = (s.ptr - base) // (e * ld)
                assert (s.ptr - base) % (e * ld) == 0 and s.row0 == r0 and s.ld == ld and s.cols == hidden
                assert np.array_equal(full[r0:r0 + s.rows, :hidden], rs)
        else:
            rows, cols = int(rng.integers(1, 33)), int(rng.integers(1, 33))
            ld = cols + int(rng.integers(0, 3))
            full = np.arange(rows * ld).reshape(rows, ld)
            fn = W.view_col if kind == F.KV_W_COLUMN else W.view_row
            try:
                (ref,) = fn(full[:, :cols], r, m)
            except (W.RankOutOfRange, W.IndivisibleExtent):
                with pytest.raises(F.FlyKVError):
                    F.weight_shard_view(F.weight_desc(base, rows, cols, e, kind, ld=ld), r, m)
                continue
            s = F.weight_shard_view(F.weight_desc(base, rows, cols, e, kind, ld=ld), r, m).seg[0]
            off = s.ptr - base
            assert off % e == 0 and s.ld == ld
            r0, c0 = divmod(off // e, ld)
            assert (s.row0, s.col0) == (r0, c0)
            assert np.array_equal(full[r0:r0 + s.rows, c0:c0 + s.cols], ref)


def test_suggested_rank_ids_are_optimal_by_brute_force():
    """N2 pin: kv_suggest_rank_ids' assignment keeps as many bytes local as
    the best of all p! rank-ID permutations of the destination group, with
    the local bytes of each permutation counted from the oracle's atom map
    (random sources of every degree, random source rank IDs, p = 2 and 4)."""
    import itertools
    rng = np.random.default_rng(77)
    for case in range(30):
        H = int(rng.choice([1, 2, 4, 8]))
        geo = (1, H, 8, 4, 2)
        og = O.Geom(*geo)
        p = int(rng.choice([2, 4]))
        dst = (int(rng.integers(0, 8 // p)) * p, p)
        c = fake_cache(geo, [512] * 8)
        mirror = [np.zeros(512, dtype=np.uint8) for _ in range(8)]
        degs = [q for q in (1, 2, 4, 8) if (q <= H and H % q == 0) or (q > H and q % H == 0)]
        if not ((p <= H and H % p == 0) or (p > H and p % H == 0)):
            continue
        reqs = []
        for i in range(int(rng.integers(1, 5))):
            q = int(rng.choice(degs))
            src = (int(rng.integers(0, 8 // q)) * q, q)
            T = int(rng.integers(1, 90))
            srid = [int(x) for x in rng.permutation(q)] if q > 1 and rng.random() < 0.5 else None
            reqs.append((i, T, src, oracle_alloc(c, mirror, src, O.num_blocks(og, T, q)), dst, srid))
        sugg = F.kv_suggest_rank_ids(c, reqs, dst)

        def local_bytes(rid):
            tot = 0
            for (_, T, s, ids, d, srid) in reqs:
                tab1 = list(range(O.num_blocks(og, T, d[1])))          # IDs do not matter for locality
                sg, _, dg, _ = O.atom_map(og, [512] * 8, T, s, list(ids), d, tab1, srid, rid)
                tot += int((sg == dg).sum())
            return tot
        best = max(local_bytes(list(perm)) for perm in itertools.permutations(range(p)))
        assert local_bytes(sugg) == best, (case, sugg)


def test_paged_decode_validates_before_the_device():
    """kv_paged_decode argument checks need no GPU: geometry (bf16, head_dim
    64/128/256), counts, NULL pointers, 16-byte alignment of q and the layer
    base, a negative max_seq_len; n_res = 0 is a no-op."""
    g = F.geometry(2, 4, 128, 16, 2)
    a16 = 1 << 40
    args = dict(layer_base=a16, n_res=4, req_ptr=a16, block_ids=a16, per_req_meta=a16, seq_lens=a16,
                q_heads_local=8, q=a16, out=a16, scale=0.1, max_seq_len=100)

    def call(geom=g, **kw):
        d = dict(args, **kw)
        F.kv_paged_decode(geom, d["layer_base"], d["n_res"], d["req_ptr"], d["block_ids"], d["per_req_meta"],
                          d["seq_lens"], d["q_heads_local"], d["q"], d["out"], d["scale"], d["max_seq_len"])

    for geom, kw in ((F.geometry(2, 4, 96, 16, 2), {}), (F.geometry(2, 4, 128, 16, 4), {}), (g, {"n_res": -1}),
                     (g, {"q_heads_local": 0}), (g, {"req_ptr": None}), (g, {"q": a16 + 8}),
                     (g, {"layer_base": a16 + 4}), (g, {"max_seq_len": -1}), (g, {"seq_lens": None})):
        with pytest.raises(F.FlyKVError) as e:
            call(geom, **kw)
        assert e.value.name == "KV_ERR_INVALID_ARG", (geom.head_dim, kw)
    call(n_res=0)   # nothing resident: no launch, no device work
    st = F._lib.kv_paged_decode(F.C.byref(g), a16, 4, a16, a16, a16, a16, 8, a16, a16, 0.1, 100, 2, None)
    assert F.STATUS_NAMES[st] == "KV_ERR_INVALID_ARG"   # unknown flag bits
