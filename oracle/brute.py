"""Brute-force enumerator for tiny KV caches -- a second, independent oracle.

ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header).

Unlike kv_oracle.c, which computes byte offsets, this module works on the
*logical* KV tensor of every request, kv[l, kv, h, t, :] (d elements), and
reads/writes physical blocks through numpy reshapes of the block bytes into
the multi-dimensional block layout the paper describes:

    block at degree p  ==  array[2 (K/V), H_loc(p), B(p), d]       (R4)
    H_loc(p) = H // p  (p <= H)  else 1                            (Eq.3, R2)
    B(p)     = B * H // H_loc(p)                                   (Eq.2, R2)
    rank r of a degree-p group holds heads
        [r*H_loc, (r+1)*H_loc)        if p <= H                    (Eq.1, R3)
        {r // (p // H)}               if p >  H                    (GQA replication, R2)

Pure-Python loops over requests/tokens: use only on tiny caches.
"""
from __future__ import annotations

import numpy as np


def h_loc(H: int, p: int) -> int:
    return H // p if p <= H else 1


def b_of(H: int, B: int, p: int) -> int:
    return B * (H // h_loc(H, p))


def heads_of_rank(H: int, p: int, r: int) -> list:
    if p <= H:
        hl = H // p
        return list(range(r * hl, (r + 1) * hl))
    return [r // (p // H)]


def block_view(pool: np.ndarray, L: int, nb: int, M: int, l: int, blk: int,
               H: int, B: int, d: int, p: int, e: int) -> np.ndarray:
    """Writable [2, H_loc, B(p), d*e] uint8 view of one block of one layer."""
    base = (l * nb + blk) * M
    raw = pool[base:base + M]
    return raw.reshape(2, h_loc(H, p), b_of(H, B, p), d * e)


def read_request(pools, geo, group, table, T_slots, rid=None):
    """Gather the logical KV of one request: array [L, 2, H, T_slots, d*e] (uint8).

    Every replica of a head is read; an assertion checks replicas agree
    (head-ownership invariant).  rid[m] = rank ID of member m (None =
    identity): member m holds the head slice of rank ID rid[m].
    """
    L, H, d, B, e = geo
    M = 2 * H * B * d * e
    g0, p = group
    out = np.zeros((L, 2, H, T_slots, d * e), dtype=np.uint8)
    seen = np.zeros((H,), dtype=bool)
    bp = b_of(H, B, p)
    for r in range(p):
        pool = pools[g0 + r]
        nb = pool.size // (L * M)
        heads = heads_of_rank(H, p, rid[r] if rid is not None else r)
        for t in range(T_slots):
            blk = table[t // bp]
            s = t % bp
            for l in range(L):
                v = block_view(pool, L, nb, M, l, blk, H, B, d, p, e)
                for i, h in enumerate(heads):
                    if seen[h]:
                        assert np.array_equal(out[l, :, h, t], v[:, i, s]), "replicas differ"
                    else:
                        out[l, :, h, t] = v[:, i, s]
        for h in heads:
            seen[h] = True
    assert seen.all()
    return out


def write_request(pools, geo, group, table, logical, rid=None):
    """Scatter logical KV [L, 2, H, T_slots, d*e] into every owner's blocks."""
    L, H, d, B, e = geo
    M = 2 * H * B * d * e
    g0, p = group
    bp = b_of(H, B, p)
    T_slots = logical.shape[3]
    for r in range(p):
        pool = pools[g0 + r]
        nb = pool.size // (L * M)
        heads = heads_of_rank(H, p, rid[r] if rid is not None else r)
        for t in range(T_slots):
            blk = table[t // bp]
            s = t % bp
            for l in range(L):
                v = block_view(pool, L, nb, M, l, blk, H, B, d, p, e)
                for i, h in enumerate(heads):
                    v[:, i, s] = logical[l, :, h, t]


def lowest_common_free(held, group, n):
    """The n lowest block IDs free on every GPU of group (R6, R8)."""
    g0, p = group
    free = np.ones_like(held[g0], dtype=bool)
    for r in range(p):
        free &= held[g0 + r] == 0
    ids = np.nonzero(free)[0][:n]
    if len(ids) < n:
        return None
    return [int(i) for i in ids]


def switch(pools, held, geo, reqs):
    """Brute-force switch with the same contract as oracle.switch.

    reqs: objects with .T, .src (g0,p), .src_ids, .dst (g0,p).
    Returns list of destination tables, or None on out-of-blocks.
    """
    L, H, d, B, e = geo
    tabs = []

    def same(rq):  # same group and same rank IDs (R12, R19)
        a = getattr(rq, "src_rid", None) or list(range(rq.src[1]))
        b = getattr(rq, "dst_rid", None) or list(range(rq.dst[1]))
        return tuple(rq.src) == tuple(rq.dst) and list(a) == list(b)

    for rq in reqs:
        if same(rq):
            tabs.append(list(rq.src_ids))
            continue
        n1 = -(-rq.T // b_of(H, B, rq.dst[1]))
        ids = lowest_common_free(held, rq.dst, n1)
        if ids is None:
            return None
        for r in range(rq.dst[1]):
            held[rq.dst[0] + r][ids] = 1
        slots = -(-rq.T // B) * B  # whole B-token atoms (R9)
        logical = read_request(pools, geo, rq.src, rq.src_ids, slots, getattr(rq, "src_rid", None))
        write_request(pools, geo, rq.dst, ids, logical, getattr(rq, "dst_rid", None))
        tabs.append(ids)
    for rq in reqs:
        if same(rq):
            continue
        for r in range(rq.src[1]):
            held[rq.src[0] + r][list(rq.src_ids)] = 0
    return tabs
