"""Pins for the oracle (CPU only): the oracle is checked against values the
paper prints, closed forms, library routines, invariants and a second,
independent brute-force enumerator -- never against itself.

Citations: P:n = PAPER.md line, S:n = SPEC.md line, Rn = DESIGN.md reading.
"""
import os
import re

import numpy as np
import pytest

from oracle import brute
from oracle import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------ layout pins
def test_fig4_block_sizes():
    """Fig.4 caption: B_base=4 tokens in DP, 8 in 2TP, 16 in 4TP."""
    g = O.Geom(L=1, H=4, d=8, B=4, e=2)
    assert [O.block_tokens(g, p) for p in (1, 2, 4)] == [4, 8, 16]


def test_eq3_example():
    """Eq.3 with B_base=16, H_base=8, N_eng=4 -> B_req=64, H_req=2."""
    g = O.Geom(L=1, H=8, d=128, B=16, e=2)
    assert O.block_tokens(g, 4) == 64
    assert O.h_loc(g, 4) == 2


@pytest.mark.parametrize("H", [1, 2, 4, 8])
@pytest.mark.parametrize("p", [1, 2, 4, 8, 16])
def test_block_byte_invariance(H, p):
    """M_block = B(p)*D_local(p)*P_size is the same for every degree."""
    g = O.Geom(L=3, H=H, d=64, B=16, e=2)
    M = O.block_bytes(g)
    assert M == 2 * H * 16 * 64 * 2
    assert 2 * O.block_tokens(g, p) * O.h_loc(g, p) * 64 * 2 == M
    # Eq.2 holds exactly whenever p divides H
    if p <= H:
        assert O.block_tokens(g, p) == p * 16


def test_allocate_examples():
    """SPEC allocate examples: ceil(9/4)=3, ceil(9/8)=2 with B_base=4."""
    g = O.Geom(L=1, H=2, d=4, B=4, e=2)
    assert O.num_blocks(g, 9, 1) == 3
    assert O.num_blocks(g, 9, 2) == 2
    assert O.num_blocks(g, 0, 2) == 0


@pytest.mark.parametrize("L,T,expect", [(80, 1, 327680), (32, 1, 131072)])
def test_kv_bytes_per_token(L, T, expect):
    """2*L*H*d*e bytes per token (H=8, d=128, bf16)."""
    g = O.Geom(L=L, H=8, d=128, B=16, e=2)
    assert L * O.block_bytes(g) // g.B == expect


@pytest.mark.parametrize("H", [1, 2, 4, 8])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_head_ownership(H, p):
    """Every head lives on exactly max(1, p/H) ranks; ranks' head sets tile
    [0,H) contiguously (P:278 'disjoint subset', Eq.1, R2, R3)."""
    g = O.Geom(L=1, H=H, d=8, B=4, e=2)
    owners = {h: sorted(O.owner_rank(g, p, h, j) for j in range(O.replicas(g, p))) for h in range(H)}
    all_ranks = sorted(r for v in owners.values() for r in v)
    if p <= H:
        assert all(len(v) == 1 for v in owners.values())
        assert sorted(set(all_ranks)) == list(range(p))
        for r in range(p):
            hs = [h for h in range(H) if owners[h] == [r]]
            assert hs == list(range(r * H // p, (r + 1) * H // p))
            assert O.first_head(g, p, r) == hs[0]
    else:
        assert all_ranks == list(range(p))  # each rank exactly one head
        for r in range(p):
            assert O.first_head(g, p, r) == r // (p // H)
    assert O.h_loc(g, p) * min(p, H) == H


@pytest.mark.parametrize("T", [1, 15, 16, 17, 100, 4096, 4097])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_block_count_bounds(T, p):
    """ceil(T/B) <= p*ceil(T/(pB)) <= ceil(T/B) + p - 1."""
    g = O.Geom(L=1, H=8, d=8, B=16, e=2)
    c = -(-T // 16)
    n = O.num_blocks(g, T, p)
    assert c <= p * n <= c + p - 1


# ------------------------------------------------------------ golden example
def _parse_golden():
    spec = {"held": {}, "atoms": []}
    with open(os.path.join(GOLDEN, "worked_example.txt")) as f:
        for line in f:
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            k, *rest = line.split()
            if k == "geometry":
                kv = dict(x.split("=") for x in rest)
                spec["geo"] = O.Geom(**{a: int(b) for a, b in kv.items()})
            elif k == "pool_blocks":
                spec["nb"] = [int(x) for x in rest]
            elif k == "held":
                spec["held"][int(rest[0])] = [int(x) for x in rest[1:]]
            elif k == "request":
                kv = dict(x.split("=") for x in rest)
                spec["req"] = O.Req(int(kv["T"]), tuple(int(x) for x in kv["src"].split(",")),
                                    [int(x) for x in kv["table"].split(",")],
                                    tuple(int(x) for x in kv["dst"].split(",")))
            elif k == "expect_dst_table":
                spec["dst_table"] = [int(x) for x in rest]
            elif k == "atom_bytes":
                spec["atom_bytes"] = int(rest[0])
            elif k == "atom":
                kv = dict(x.split("=") for x in rest)
                sg, so = (int(x) for x in kv["src"].split(":"))
                dg, do = (int(x) for x in kv["dst"].split(":"))
                spec["atoms"].append((int(kv["kv"]), int(kv["h"]), int(kv["c"]), sg, so, dg, do))
            elif k == "untouched_block":
                a, b = re.match(r"slots=(\d+)-(\d+)", rest[1]).groups()
                spec["untouched"] = (int(rest[0]), int(a), int(b))
    return spec


def test_worked_example_golden():
    s = _parse_golden()
    g = s["geo"]
    M = O.block_bytes(g)
    rng = np.random.default_rng(0)
    pools = [rng.integers(0, 256, size=g.L * n * M, dtype=np.uint8) for n in s["nb"]]
    before = [p.copy() for p in pools]
    held = [np.zeros(n, dtype=np.uint8) for n in s["nb"]]
    for gpu, ids in s["held"].items():
        held[gpu][ids] = 1
    st, tabs = O.switch(g, pools, held, [s["req"]])
    assert st == 0
    assert list(tabs[0]) == s["dst_table"]
    ab = s["atom_bytes"]
    assert ab == g.B * g.d * g.e
    for (kv, h, c, sg, so, dg, do) in s["atoms"]:
        # the oracle's own locate agrees with the hand-computed offsets
        assert O.locate(g, 0, 1, s["req"].src_ids, kv, h, c * g.B) == (sg, so)
        assert O.locate(g, 0, 2, tabs[0], kv, h, c * g.B) == (dg, do)
        for l in range(g.L):
            sl = l * s["nb"][sg] * M
            dl = l * s["nb"][dg] * M
            assert np.array_equal(pools[dg][dl + do:dl + do + ab], before[sg][sl + so:sl + so + ab])
    blk, s0, s1 = s["untouched"]
    bp = O.block_tokens(g, 2)
    row = g.d * g.e
    for gpu in (0, 1):
        for l in range(g.L):
            for kv in range(2):
                for hl in range(O.h_loc(g, 2)):
                    base = (l * s["nb"][gpu] + blk) * M + kv * M // 2 + hl * bp * row
                    a, b = base + s0 * row, base + (s1 + 1) * row
                    assert np.array_equal(pools[gpu][a:b], before[gpu][a:b])
    # source IDs released, destination IDs held on both ranks
    assert sorted(np.nonzero(held[0])[0]) == [1, 4]
    assert sorted(np.nonzero(held[1])[0]) == [0, 1, 3, 4]


# ------------------------------------------------------------ helpers
def _setup(geo, nb, reqs_spec, seed):
    """Random pools, held sets from the requests' source tables."""
    g = O.Geom(*geo)
    M = O.block_bytes(g)
    rng = np.random.default_rng(seed)
    pools = [rng.integers(0, 256, size=g.L * n * M, dtype=np.uint8) for n in nb]
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    reqs = []
    perms = {}
    for (T, src, dst) in reqs_spec:
        n = O.num_blocks(g, T, src[1])
        if src not in perms:
            perms[src] = list(rng.permutation(min(nb[x] for x in range(src[0], src[0] + src[1]))))
        ids = [int(perms[src].pop()) for _ in range(n)]
        for r in range(src[1]):
            held[src[0] + r][ids] = 1
        if src[1] > g.H:  # GQA replicas start byte-identical (R2, R10)
            rep = src[1] // g.H
            for r in range(src[1]):
                lo = src[0] + (r // rep) * rep
                for l in range(g.L):
                    for b in ids:
                        a = (l * nb[lo] + b) * M
                        z = (l * nb[src[0] + r] + b) * M
                        pools[src[0] + r][z:z + M] = pools[lo][a:a + M]
        reqs.append(O.Req(T, src, ids, dst))
    return g, pools, held, reqs


GRID_T = [1, 5, 16, 17, 31, 32, 33, 64, 70]


def _grid():
    cases = []
    for H in (1, 2, 4):
        for p0 in (1, 2, 4):
            for p1 in (1, 2, 4):
                cases.append((H, p0, p1))
    return cases


@pytest.mark.parametrize("H,p0,p1", _grid())
def test_c_oracle_matches_brute_force(H, p0, p1):
    """Independent brute-force enumerator (logical tensor + numpy block
    reshapes) and the C oracle (byte offsets) agree on every byte of every
    pool, on destination tables and on the allocator state."""
    geo = (2, H, 4, 4, 2)  # L, H, d, B, e
    n_gpus = 4
    nb = [256] * n_gpus
    rng = np.random.default_rng(H * 100 + p0 * 10 + p1)
    spec = []
    for i, T in enumerate(GRID_T):
        src = ((i * p0) % n_gpus // p0 * p0, p0)
        dst = ((i * p1 + p1) % n_gpus // p1 * p1, p1)
        spec.append((T + int(rng.integers(0, 3)), src, dst))
    g, pools, held, reqs = _setup(geo, nb, spec, seed=7)
    pools_b = [p.copy() for p in pools]
    held_b = [h.copy() for h in held]
    st, tabs = O.switch(g, pools, held, reqs)
    tabs_b = brute.switch(pools_b, held_b, geo, reqs)
    assert st == 0 and tabs_b is not None
    assert [list(t) for t in tabs] == [list(t) for t in tabs_b]
    for a, b in zip(pools, pools_b):
        assert np.array_equal(a, b)
    for a, b in zip(held, held_b):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("H", [1, 2, 4, 8])
@pytest.mark.parametrize("p0,p1", [(1, 2), (1, 4), (1, 8), (2, 1), (4, 2), (8, 1), (2, 8), (8, 2), (4, 8)])
def test_round_trip_identity(H, p0, p1):
    """X -> Y -> X restores every request's logical KV (SURVEY 8(c) round trip),
    including GQA replication (p > H); checked through the brute-force reader."""
    geo = (2, H, 4, 4, 2)
    n_gpus = 8
    nb = [160] * n_gpus
    Ts = [1, 7, 16, 33, 64, 90]
    spec = []
    for i, T in enumerate(Ts):
        spec.append((T, ((i * p0) % n_gpus, p0), ((i * p1) % n_gpus, p1)))
    g, pools, held, reqs = _setup(geo, nb, spec, seed=H + 31 * p0 + 7 * p1)
    slots = [-(-T // 4) * 4 for T in Ts]
    before = [brute.read_request(pools, geo, r.src, r.src_ids, s) for r, s in zip(reqs, slots)]
    held0 = sum(int(h.sum()) for h in held)
    st, tabs = O.switch(g, pools, held, reqs)
    assert st == 0
    mid = [brute.read_request(pools, geo, r.dst, t, s) for r, t, s in zip(reqs, tabs, slots)]
    for a, b in zip(before, mid):
        assert np.array_equal(a, b)
    back = [O.Req(r.T, r.dst, list(t), r.src) for r, t in zip(reqs, tabs)]
    st, tabs2 = O.switch(g, pools, held, back)
    assert st == 0
    after = [brute.read_request(pools, geo, r.src, t, s) for r, t, s in zip(reqs, tabs2, slots)]
    for a, b in zip(before, after):
        assert np.array_equal(a, b)
    # pool conservation: same number of held blocks as at the start
    assert sum(int(h.sum()) for h in held) == held0


@pytest.mark.parametrize("H,p", [(4, 2), (8, 4), (8, 8), (2, 2), (4, 4)])
def test_closed_form_permute(H, p):
    """DP -> TP_p with a contiguous source table and p*B | T equals the numpy
    reshape/transpose  src.reshape(L,J,p,2,p,H/p,B,d).transpose(4,0,1,3,5,2,6,7)
    (SURVEY 8(c) closed form; the library routine is the reference)."""
    L, d, B, e = 3, 8, 4, 2
    T = p * B * 5
    J = T // (p * B)
    C = T // B
    g = O.Geom(L, H, d, B, e)
    M = O.block_bytes(g)
    nb = C + J + 4
    rng = np.random.default_rng(H * p)
    pools = [rng.integers(0, 256, size=L * nb * M, dtype=np.uint8) for _ in range(p)]
    held = [np.zeros(nb, dtype=np.uint8) for _ in range(p)]
    held[0][:C] = 1
    src = pools[0].reshape(L, nb, M)[:, :C].copy()  # [L, C, M]
    st, tabs = O.switch(g, pools, held, [O.Req(T, (0, 1), list(range(C)), (0, p))])
    assert st == 0
    assert list(tabs[0]) == list(range(C, C + J))  # lowest free on all ranks
    ref = src.reshape(L, C, 2, H, B, d * e).reshape(L, J, p, 2, p, H // p, B, d * e)
    ref = ref.transpose(4, 0, 1, 3, 5, 2, 6, 7)  # [r, L, J, 2, H/p, p(q), B, d*e]
    for r in range(p):
        got = pools[r].reshape(L, nb, M)[:, C:C + J].reshape(L, J, 2, H // p, p, B, d * e)
        assert np.array_equal(got, ref[r])


def test_only_destination_atoms_change():
    """Bytes outside the destination atoms are untouched (poison survives,
    requests absent from the plan unchanged, P:575 hard-preempt coexistence)."""
    geo = (2, 4, 8, 4, 2)
    g, pools, held, reqs = _setup(geo, [40, 40], [(10, (0, 1), (0, 2)), (33, (1, 1), (0, 2)),
                                                   (5, (0, 1), (0, 1))], seed=3)
    before = [p.copy() for p in pools]
    st, tabs = O.switch(g, pools, held, reqs)
    assert st == 0
    M = O.block_bytes(g)
    atom = g.B * g.d * g.e
    allowed = [np.zeros(p.size, dtype=bool) for p in pools]
    for r, t in zip(reqs, tabs):
        if r.src == r.dst:
            continue
        for l in range(g.L):
            for kv in range(2):
                for h in range(g.H):
                    for c in range(-(-r.T // g.B)):
                        for j in range(O.replicas(g, r.dst[1])):
                            gpu, off = O.locate(g, r.dst[0], r.dst[1], t, kv, h, c * g.B, j)
                            base = l * (pools[gpu].size // (g.L * M)) * M + off
                            allowed[gpu][base:base + atom] = True
    for a, b, m in zip(pools, before, allowed):
        changed = a != b
        assert not np.any(changed & ~m)


def test_out_of_blocks():
    g, pools, held, reqs = _setup((1, 2, 4, 4, 2), [4, 4], [(12, (0, 1), (0, 2))], seed=1)
    # source holds 3 of 4 blocks on GPU0 -> only 1 common free ID, need 2
    st, _ = O.switch(g, pools, held, reqs)
    assert st == 6


def test_tables_csr():
    """Per-GPU tables list exactly the requests resident on that GPU, in
    request order, with capacity B(p), H_loc and first head."""
    geo = (1, 8, 4, 4, 2)
    g, pools, held, reqs = _setup(geo, [64] * 4, [(40, (0, 1), (0, 2)), (9, (1, 1), (0, 4)),
                                                  (17, (2, 1), (2, 2)), (3, (3, 1), (3, 1))], seed=5)
    st, tabs = O.switch(g, pools, held, reqs)
    assert st == 0
    rp, ids, meta = O.tables(g, 1, reqs, tabs)
    assert list(meta[:, 0]) == [0, 1]
    assert list(meta[0, 1:]) == [8, 4, 4]     # TP2: B(2)=8, H_loc=4, rank1 starts at head 4
    assert list(meta[1, 1:]) == [16, 2, 2]    # TP4: B(4)=16, H_loc=2, rank1 starts at head 2
    assert list(ids) == list(tabs[0]) + list(tabs[1])
    assert list(rp) == [0, len(tabs[0]), len(tabs[0]) + len(tabs[1])]
    rp3, ids3, meta3 = O.tables(g, 3, reqs, tabs)
    assert list(meta3[:, 0]) == [1, 2, 3] and list(meta3[2, 1:]) == [4, 8, 0]


def test_atom_map_matches_switch():
    """or_atom_map enumerates exactly the bytes or_switch moves: applying the
    map with numpy copies reproduces the oracle's pools."""
    geo = (2, 4, 8, 4, 2)
    g, pools, held, reqs = _setup(geo, [64] * 8, [(37, (0, 1), (0, 2)), (9, (2, 2), (0, 8)), (70, (4, 4), (4, 1))],
                                  seed=12)
    before = [p.copy() for p in pools]
    mine = [p.copy() for p in pools]
    st, tabs = O.switch(g, pools, held, reqs)
    assert st == 0
    atom = g.B * g.d * g.e
    for r, t in zip(reqs, tabs):
        sg, so, dg, do = O.atom_map(g, [64] * 8, r.T, r.src, r.src_ids, r.dst, t)
        for a, b, c, d in zip(sg, so, dg, do):
            mine[c][d:d + atom] = before[a][b:b + atom]
    for a, b in zip(mine, pools):
        assert np.array_equal(a, b)


# ------------------------------------------------------------ rank-ID assignment (N2)
def _perm(rng, p):
    return [int(x) for x in rng.permutation(p)]


@pytest.mark.parametrize("H,p0,p1", [(4, 1, 2), (4, 2, 4), (4, 4, 2), (2, 1, 4), (2, 4, 1), (1, 2, 4), (4, 4, 4)])
def test_rank_ids_c_oracle_matches_brute(H, p0, p1):
    """Rank-ID assignments (member m holds rank ID rid[m]'s slice):
    the C oracle and the brute-force enumerator agree for random
    permutations on both sides; replicated sources are made consistent
    under their own rank IDs first."""
    rng = np.random.default_rng(H * 13 + p0 * 7 + p1)
    geo = (2, H, 4, 4, 2)
    g = O.Geom(*geo)
    M = O.block_bytes(g)
    n_gpus = 4
    nb = [256] * n_gpus
    spec = [(T, ((i * p0) % n_gpus // p0 * p0, p0), (((i + 1) * p1) % n_gpus // p1 * p1, p1))
            for i, T in enumerate([1, 17, 33, 64, 70])]
    g_, pools, held, reqs = _setup(geo, nb, spec, seed=3)
    for r in reqs:
        r.src_rid = _perm(rng, r.src[1])
        r.dst_rid = _perm(rng, r.dst[1]) if tuple(r.dst) != tuple(r.src) else r.src_rid
        if r.src[1] > H:  # replicas identical under the source rank IDs
            rep = r.src[1] // H
            for m in range(r.src[1]):
                lo = r.src_rid.index((r.src_rid[m] // rep) * rep)
                for l in range(g.L):
                    for b in r.src_ids:
                        a = (l * nb[r.src[0] + lo] + b) * M
                        z = (l * nb[r.src[0] + m] + b) * M
                        pools[r.src[0] + m][z:z + M] = pools[r.src[0] + lo][a:a + M]
    pools_b = [p.copy() for p in pools]
    held_b = [h.copy() for h in held]
    st, tabs = O.switch(g, pools, held, reqs)
    tabs_b = brute.switch(pools_b, held_b, geo, reqs)
    assert st == 0 and [list(t) for t in tabs] == [list(t) for t in tabs_b]
    for a, b in zip(pools, pools_b):
        assert np.array_equal(a, b)


def test_rank_ids_identity_and_round_trip():
    """rid = identity reproduces the default layout (R3) byte for byte, and a
    permuted TP4 -> TP8 -> permuted TP4 round trip restores the logical KV."""
    geo = (2, 8, 4, 4, 2)
    g = O.Geom(*geo)
    spec = [(T, (0, 4), (0, 8)) for T in (5, 64, 131)]
    _, p1, h1, r1 = _setup(geo, [128] * 8, spec, seed=4)
    _, p2, h2, r2 = _setup(geo, [128] * 8, spec, seed=4)
    for r in r2:
        r.src_rid, r.dst_rid = [0, 1, 2, 3], list(range(8))
    assert O.switch(g, p1, h1, r1)[0] == 0 and O.switch(g, p2, h2, r2)[0] == 0
    assert all(np.array_equal(a, b) for a, b in zip(p1, p2))
    _, pools, held, reqs = _setup(geo, [128] * 8, spec, seed=5)
    for r in reqs:
        r.src_rid = [2, 0, 3, 1]
        r.dst_rid = [0, 2, 4, 6, 1, 3, 5, 7]
    slots = [-(-r.T // 4) * 4 for r in reqs]
    before = [brute.read_request(pools, geo, r.src, r.src_ids, s, r.src_rid) for r, s in zip(reqs, slots)]
    st, tabs = O.switch(g, pools, held, reqs)
    assert st == 0
    back = [O.Req(r.T, r.dst, list(t), r.src, r.dst_rid, r.src_rid) for r, t in zip(reqs, tabs)]
    st, tabs2 = O.switch(g, pools, held, back)
    assert st == 0
    after = [brute.read_request(pools, geo, r.src, t, s, r.src_rid) for r, t, s in zip(reqs, tabs2, slots)]
    assert all(np.array_equal(a, b) for a, b in zip(before, after))


def test_rank_ids_keep_heads_local():
    """N2: promoting TP4 -> TP8 with rank IDs [0,2,4,6,1,3,5,7] keeps one of
    each source GPU's two heads on that GPU: half the atoms stay local,
    against 1/8 with the identity assignment."""
    g = O.Geom(2, 8, 4, 4, 2)
    _, pools, held, reqs = _setup((2, 8, 4, 4, 2), [128] * 8, [(64, (0, 4), (0, 8))], seed=6)
    r = reqs[0]
    tab1 = list(range(100, 100 + O.num_blocks(g, 64, 8)))
    for rid, want in ((None, 1 / 8), ([0, 2, 4, 6, 1, 3, 5, 7], 1 / 2)):
        sg, so, dg, do = O.atom_map(g, [128] * 8, 64, (0, 4), r.src_ids, (0, 8), tab1, None, rid)
        assert np.mean(sg == dg) == pytest.approx(want)


def test_same_group_repermutation_moves():
    """R19: staying in the same TP4 group with new rank IDs moves every head
    whose owner changes; brute force and the C oracle agree."""
    geo = (2, 8, 4, 4, 2)
    g = O.Geom(*geo)
    _, pools, held, reqs = _setup(geo, [64] * 4, [(40, (0, 4), (0, 4)), (9, (0, 4), (0, 4))], seed=8)
    for r in reqs:
        r.src_rid, r.dst_rid = [0, 1, 2, 3], [1, 0, 3, 2]
    pools_b = [p.copy() for p in pools]
    held_b = [h.copy() for h in held]
    st, tabs = O.switch(g, pools, held, reqs)
    tabs_b = brute.switch(pools_b, held_b, geo, reqs)
    assert st == 0 and [list(t) for t in tabs] == [list(t) for t in tabs_b]
    assert all(set(t).isdisjoint(r.src_ids) for t, r in zip(tabs, reqs))  # fresh blocks
    assert all(np.array_equal(a, b) for a, b in zip(pools, pools_b))


@pytest.mark.parametrize("H,p0,p1,T", [(4, 1, 4, 90), (4, 4, 1, 77), (2, 2, 8, 65), (4, 2, 4, 100), (8, 8, 2, 50)])
def test_pieces_concatenate_to_the_whole_request(H, p0, p1, T):
    """R20 pinned by brute force: moving a request as consecutive pieces cut
    on whole blocks of both layouts (each a plain request on its slice of the
    source table, one oracle switch per piece with sources released between)
    leaves, under the concatenated destination table, exactly the logical KV
    of the request (brute.read_request), as the one-shot move does."""
    geo = (2, H, 4, 4, 2)
    g = O.Geom(*geo)
    nb = [120] * 8
    g_, pools, held, reqs = _setup(geo, nb, [(T, (0, p0), (0, p1))], seed=H * 7 + p0 + p1)
    r = reqs[0]
    slots = -(-T // 4) * 4
    before = brute.read_request(pools, geo, r.src, r.src_ids, slots)
    b0, b1 = O.block_tokens(g, p0), O.block_tokens(g, p1)
    unit = max(b0, b1)
    cuts = [0] + [c for c in range(unit, T, 2 * unit)] + [T]   # pieces of 2 units, ragged last
    parts = []
    for t0, t1 in zip(cuts, cuts[1:]):
        piece = O.Req(t1 - t0, r.src, list(r.src_ids[t0 // b0: -(-t1 // b0)]), r.dst)
        st, tabs = O.switch(g, pools, held, [piece])
        assert st == 0
        parts += list(tabs[0])
    assert len(parts) == O.num_blocks(g, T, p1)
    after = brute.read_request(pools, geo, r.dst, parts, slots)
    assert np.array_equal(before, after)
