"""Consumer proof: the re-laid-out cache is usable.

Paged decode attention (kv_paged_decode, sm_100a) reads each pool through the
CSR tables and per-request (B(p), H_loc, first head) that
kv_remap_block_tables produces -- the "stride and capacity" the paper's
Adaptor passes to the attention kernel.  On synthetic Q and finite
bf16 KV:
  * the DP replica's output matches an fp64 numpy attention (the oracle's
    locate() gives each token's bytes) within fp32 tolerance, for every
    request and every query head;
  * after DP -> TP (incl. GQA replication, TP > kv_heads), every TP rank's
    output for its query heads (the Eq.1 column slice of Q) is bit-identical
    to the DP output for the same heads, and within the same tolerance of
    the fp64 oracle.
"""
import numpy as np
import pytest

import synth
from oracle import oracle as O
from oracle.attention import decode_attention

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _decode_all(F, eng, geo, plan, tables, q_full, gpus, q_slices, seq):
    """Run decode on each GPU's table; returns {(plan_index, global_q_head): out row}."""
    L, H, d, B, e = geo
    M = F.kv_layout(eng.geom, 1)[2]
    res = {}
    for g in gpus:
        n_res, n_ids = plan.resident(g)
        if n_res == 0:
            continue
        t = tables[g]
        meta = t.meta[:n_res].cpu().numpy()
        qlo, qhi = q_slices(g, meta)
        idx = torch.as_tensor(meta[:, 0].astype(np.int64), device="cuda:0")
        q = q_full[idx, qlo:qhi].contiguous()
        lens = torch.as_tensor([seq[i] for i in meta[:, 0]], dtype=torch.int32, device="cuda:0")
        out = torch.empty((n_res, qhi - qlo, d), dtype=torch.float32, device="cuda:0")
        layer = eng.pools.tensors[g][1]  # layer 1 of pool g
        F.kv_paged_decode(eng.geom, layer.data_ptr(), n_res, t.req_ptr, t.block_ids, t.meta, lens, qhi - qlo, q, out,
                          1.0 / np.sqrt(d), max(seq), eng.stream, after_decode=True)   # after our own kernels only
        torch.cuda.synchronize()
        o = out.cpu().numpy()
        for k, i in enumerate(meta[:, 0]):
            for jj in range(qhi - qlo):
                res[(int(i), qlo + jj)] = o[k, jj]
    return res


@pytest.mark.parametrize("H,Hq,p1,permuted,long", [(8, 32, 2, False, False), (8, 32, 4, False, False),
                                                    (8, 64, 8, False, False), (4, 32, 8, False, False),
                                                    (2, 16, 8, False, False), (8, 8, 2, False, False),
                                                    (8, 32, 4, True, False), (4, 32, 8, True, False),
                                                    (8, 64, 8, False, True), (2, 40, 8, True, True),
                                                    (4, 8, 8, False, True)])
def test_tp_after_relayout_equals_dp(H, Hq, p1, permuted, long):
    """long: lengths up to 1700 tokens (several 512-token splits, folded by
    the last-arriving CTA), plus an empty request (zeros); Hq = 40 over
    H = 2 gives 20 query heads per KV head (three head tiles, the last
    partial) on the DP replica and 5 per rank at TP8."""
    F = pytest.importorskip("paper_2602_22593_b200.flykv")
    from paper_2602_22593_b200.engine import KVSwitchEngine
    geo = (2, H, 128, 16, 2)
    og = O.Geom(*geo)
    n_gpus = 8
    rng = np.random.default_rng(H * 100 + Hq + p1)
    seq = [int(x) for x in rng.integers(1, 300, size=10)]
    if long:
        seq = [int(x) for x in rng.integers(1, 1700, size=10)]
        seq[3] = 0
        seq[5] = 512   # exactly one split
        seq[6] = 1025  # three splits, the last with one token
    src = [((i % n_gpus), 1) for i in range(len(seq))]
    dst = [((i * p1) % n_gpus // p1 * p1, p1) for i in range(len(seq))]
    w = synth.Workload("c", *geo, n_gpus, seq, src, dst)
    nb = synth.pool_blocks(w, slack=1.3)
    eng = KVSwitchEngine(F.geometry(*geo), nb, "cuda:0")
    gen = torch.Generator(device="cuda:0").manual_seed(int(H + Hq + p1))
    for t in eng.pools.tensors:  # finite bf16 contents
        t.view(torch.bfloat16).copy_(torch.randn(t.numel() // 2, generator=gen, device="cuda:0").view(t.shape[0], t.shape[1], -1))
    counts = [O.num_blocks(og, T, s[1]) for T, s in zip(seq, src)]
    tabs0 = synth.source_tables(w, counts, nb)
    for s_, ids in zip(src, tabs0):
        eng.cache.reserve(s_, ids)
    q_full = torch.randn((len(seq), Hq, 128), generator=gen, device="cuda:0").to(torch.bfloat16)
    # DP tables via a no-op plan (src == dst keeps the table, remap lists it)
    noop = [(i, T, s_, ids, s_) for i, (T, s_, ids) in enumerate(zip(seq, src, tabs0))]
    plan_dp, tables_dp, _ = eng.switch(noop, read_back=True)
    out_dp = _decode_all(F, eng, geo, plan_dp, tables_dp, q_full, range(n_gpus), lambda g, meta: (0, Hq), seq)
    # fp64 oracle on the DP layout (layer 1)
    host = [t.view(torch.int16).cpu().numpy().reshape(-1).view(np.uint16) for t in eng.pools.tensors]
    M = O.block_bytes(og)

    def bf16_to_f64(u16):
        return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)

    qf = q_full.float().cpu().numpy().astype(np.float64)
    G = Hq // H
    ref = {}
    for i in range(len(seq)):          # every request, every KV head, every query head (fp64)
        T = seq[i]
        for h in range(H):
            K = np.zeros((T, 128))
            V = np.zeros((T, 128))
            for t_ in range(T):
                gpu, off = O.locate(og, src[i][0], 1, tabs0[i], 0, h, t_)
                base = (1 * nb[gpu] * M + off) // 2
                K[t_] = bf16_to_f64(host[gpu][base:base + 128])
                gpu, off = O.locate(og, src[i][0], 1, tabs0[i], 1, h, t_)
                base = (1 * nb[gpu] * M + off) // 2
                V[t_] = bf16_to_f64(host[gpu][base:base + 128])
            for qh in range(h * G, (h + 1) * G):   # no tokens: the kernel's documented zeros
                ref[(i, qh)] = (decode_attention(K, V, qf[i, qh], 1.0 / np.sqrt(128)) if T else np.zeros(128))
    assert set(ref) == set(out_dp)
    for k, r in ref.items():
        assert np.allclose(out_dp[k], r, rtol=2e-3, atol=2e-3), k
    # switch DP -> TP_p1 and decode on every rank with its Eq.1 Q slice
    # rank IDs of the destination members: identity or a permutation;
    # member m then takes the Eq.1 Q slice of its rank ID
    rid = [int(x) for x in np.random.default_rng(p1).permutation(p1)] if permuted else list(range(p1))
    move = [(i, T, s_, ids, d_, None, rid) for i, (T, s_, ids, d_) in enumerate(zip(seq, src, tabs0, dst))]
    plan_tp, tables_tp, _ = eng.switch(move, read_back=True)
    ql = Hq // p1

    def q_slice(g, meta):
        r = rid[g % p1]  # rank ID of this member of its aligned group
        return r * ql, (r + 1) * ql
    out_tp = _decode_all(F, eng, geo, plan_tp, tables_tp, q_full, range(n_gpus), q_slice, seq)
    assert set(out_tp) == set(out_dp)
    for k, v in out_dp.items():
        assert np.array_equal(out_tp[k], v), k
        assert np.allclose(out_tp[k], ref[k], rtol=2e-3, atol=2e-3), k   # and the fp64 oracle, directly


def test_decode_workspace_not_grown_inside_graph_capture():
    """kv_paged_decode under CUDA graph capture: a workspace that would have
    to grow is refused (KV_ERR_BAD_STATE, nothing captured) -- a graph-owned
    buffer must not outlive its graph; after one call outside capture the
    same call captures and replays."""
    F = pytest.importorskip("paper_2602_22593_b200.flykv")
    g = F.geometry(1, 1, 128, 16, 2)
    dev = "cuda:0"
    layer = torch.zeros(4 * 2 * 16 * 128, dtype=torch.bfloat16, device=dev)      # 4 blocks, 1 head
    rp = torch.tensor([0, 2], dtype=torch.int32, device=dev)
    ids = torch.tensor([1, 3], dtype=torch.int32, device=dev)
    meta = torch.tensor([[0, 16, 1, 0]], dtype=torch.int32, device=dev)
    lens = torch.tensor([20], dtype=torch.int32, device=dev)
    q = torch.randn((1, 2, 128), device=dev).to(torch.bfloat16)
    out = torch.empty((1, 2, 128), dtype=torch.float32, device=dev)
    s = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with pytest.raises(F.FlyKVError) as e:
        with torch.cuda.graph(graph, stream=s):
            F.kv_paged_decode(g, layer.data_ptr(), 1, rp, ids, meta, lens, 2, q, out, 0.1, 32, s)
    assert e.value.name == "KV_ERR_BAD_STATE"
    F.kv_paged_decode(g, layer.data_ptr(), 1, rp, ids, meta, lens, 2, q, out, 0.1, 32, s)   # sizes the workspace
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        F.kv_paged_decode(g, layer.data_ptr(), 1, rp, ids, meta, lens, 2, q, out, 0.1, 32, s)
    out.fill_(7.0)
    graph.replay()
    torch.cuda.synchronize()
    assert torch.all(out == 0)   # zero K/V: every score equal, output = mean of zero V rows
    del graph
    F.kv_paged_decode_release(s)   # workspace freed; the next call on the stream allocates a new one
    F.kv_paged_decode_release(s)   # none left: a no-op
    out.fill_(7.0)
    F.kv_paged_decode(g, layer.data_ptr(), 1, rp, ids, meta, lens, 2, q, out, 0.1, 32, s)
    s.synchronize()
    assert torch.all(out == 0)


@pytest.mark.parametrize("case", list(range(36)) + ["long"])
def test_decode_random_geometry_against_fp64(case):
    """kv_paged_decode on random geometries straight from a pool: head_dim
    64/128/256, block_base 8/16/32 (B(p) not a multiple of 16 takes the
    per-row table lookup), degrees with and without GQA replication, 1-16
    query heads per KV head, lengths 0-1300 (several 512-token splits),
    random block IDs.  Member 0 of the group reads its heads; every
    (request, query head) equals fp64 attention over the tokens
    oracle.locate places, within fp32 tolerance."""
    F = pytest.importorskip("paper_2602_22593_b200.flykv")
    long = case == "long"   # 20,000 and 8,193 tokens: 40 and 17 splits, two fold levels (groups of 16)
    rng = np.random.default_rng(7100 + (99 if long else case))
    d = int(rng.choice([64, 128, 256]))
    B = int(rng.choice([8, 16, 32]))
    H = int(rng.choice([1, 2, 4, 8]))
    p = int(rng.choice([p_ for p_ in (1, 2, 4, 8) if (p_ <= H and H % p_ == 0) or (p_ > H and p_ % H == 0)]))
    og = O.Geom(1, H, d, B, 2)
    hloc = H // p if p <= H else 1
    Bp = B * H // hloc
    G = int(rng.choice([1, 2, 3, 8, 16]))
    q_local = hloc * G
    n_req = int(rng.integers(1, 7))
    seq = [int(x) for x in rng.integers(0, 1300, size=n_req)]
    if long:
        d, B, H, p, G = 128, 16, 1, 1, 2
        og = O.Geom(1, H, d, B, 2)
        hloc, Bp, q_local, n_req, seq = 1, B, 2, 3, [20000, 8193, 700]
    elif case % 5 == 0:
        seq[0] = 0
    counts = [O.num_blocks(og, T, p) for T in seq]
    M = O.block_bytes(og)
    nb = sum(counts) + 3
    perm = [int(x) for x in rng.permutation(nb)]
    tabs, k = [], 0
    for c in counts:
        tabs.append(perm[k:k + c])
        k += c
    pool = torch.randn(nb * M // 2, device="cuda:0").to(torch.bfloat16)   # finite contents everywhere
    host = pool.view(torch.int16).cpu().numpy().view(np.uint16)
    rp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    ids = np.concatenate([np.asarray(t, dtype=np.int32) for t in tabs] + [np.zeros(0, np.int32)])
    first_head = 0                                                          # member 0 of the group
    meta = np.array([[i, Bp, hloc, first_head] for i in range(n_req)], dtype=np.int32)
    dev = lambda a: torch.as_tensor(a, device="cuda:0")                     # noqa: E731
    q = torch.randn((n_req, q_local, d), device="cuda:0").to(torch.bfloat16)
    out = torch.empty((n_req, q_local, d), dtype=torch.float32, device="cuda:0")
    scale = 1.0 / np.sqrt(d)
    F.kv_paged_decode(F.geometry(1, H, d, B, 2), pool.data_ptr(), n_req, dev(rp), dev(ids) if ids.size else None,
                      dev(meta), dev(np.asarray(seq, np.int32)), q_local, q, out, scale, max(max(seq), 1))
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    qf = q.float().cpu().numpy().astype(np.float64)

    def bf(u16):
        return (u16.astype(np.uint32) << 16).view(np.float32).astype(np.float64)

    for i, T in enumerate(seq):
        for hl in range(hloc):
            h = hl if p <= H else 0          # member 0's heads: [0, H_loc), or head 0 under replication
            K = np.zeros((T, d))
            V = np.zeros((T, d))
            for t_ in range(T):
                g_, off = O.locate(og, 0, p, tabs[i], 0, h, t_)
                assert g_ == 0
                K[t_] = bf(host[off // 2:off // 2 + d])
                _, off = O.locate(og, 0, p, tabs[i], 1, h, t_)
                V[t_] = bf(host[off // 2:off // 2 + d])
            for j in range(hl * G, (hl + 1) * G):
                ref = decode_attention(K, V, qf[i, j], scale) if T else np.zeros(d)
                assert np.allclose(o[i, j], ref, rtol=2e-3, atol=2e-3), (case, i, j)


@pytest.mark.parametrize("d", [64, 128, 256])
def test_decode_back_to_back_launches_same_out(d):
    """Consecutive kv_paged_decode launches on one stream with
    KV_DECODE_AFTER_DECODE overlap through programmatic dependent launch; a
    launch's tiles may run under the previous one's tail, but its workspace
    and out writes wait for it.  Two
    launches with different q into the same out (and a third with a longer
    length bound's workspace) leave exactly the last launch's result."""
    F = pytest.importorskip("paper_2602_22593_b200.flykv")
    rng = np.random.default_rng(77)
    g = F.geometry(1, 2, d, 16, 2)
    og = O.Geom(1, 2, d, 16, 2)
    seq = [1500, 700, 33, 2600]
    counts = [O.num_blocks(og, T, 1) for T in seq]
    M = O.block_bytes(og)
    nb = sum(counts) + 2
    perm = [int(x) for x in rng.permutation(nb)]
    rp = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    ids = np.asarray(perm[:sum(counts)], dtype=np.int32)
    meta = np.array([[i, 16, 2, 0] for i in range(len(seq))], dtype=np.int32)
    dev = lambda a: torch.as_tensor(a, device="cuda:0")                     # noqa: E731
    pool = torch.randn(nb * M // 2, device="cuda:0").to(torch.bfloat16)
    lens = dev(np.asarray(seq, np.int32))
    qs = [torch.randn((len(seq), 8, d), device="cuda:0").to(torch.bfloat16) for _ in range(3)]
    s = torch.cuda.Stream()
    out = torch.empty((len(seq), 8, d), dtype=torch.float32, device="cuda:0")
    ref = torch.empty_like(out)
    args = (pool.data_ptr(), len(seq), dev(rp), dev(ids), dev(meta), lens, 8)
    for k in range(3):   # back to back on one stream, same out, overlapped (KV_DECODE_AFTER_DECODE)
        F.kv_paged_decode(g, *args, qs[k], out, 0.09, 4096 if k < 2 else 8192, s, after_decode=k > 0)
    s.synchronize()
    s2 = torch.cuda.Stream()
    F.kv_paged_decode(g, *args, qs[2], ref, 0.09, 8192, s2)
    s2.synchronize()
    assert torch.equal(out, ref)
    F.kv_paged_decode_release(s)
    F.kv_paged_decode_release(s2)
