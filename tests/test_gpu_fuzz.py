"""Randomised parity fuzz (GPU): random geometry (layers, KV heads, head_dim,
block size, element size), 2-16 virtual pools, random merges / splits /
lateral moves / no-ops with random rank-ID permutations on both sides
(incl. replicated sources and GQA destinations), random lengths incl. 0 and
tails, either kernel work order, and one of the launch paths (one launch,
per-pool launches, kv_reshard_range over a random partition of the pools,
the one-call kv_switch, pack -> all-to-all -> unpack); whole pools, tables and
allocator state bit-exact against the oracle (run_parity).  FLYKV_FUZZ_CASES
(default 24) sets the count; FLYKV_FUZZ_SEED0 the first seed."""
import os

import numpy as np
import pytest

from test_gpu_parity import run_parity

pytestmark = pytest.mark.gpu

N_CASES = int(os.environ.get("FLYKV_FUZZ_CASES", "24"))
SEED0 = int(os.environ.get("FLYKV_FUZZ_SEED0", "0"))


def _case(seed):
    rng = np.random.default_rng(50000 + seed)
    H = int(rng.choice([1, 2, 4, 8, 16]))
    d = int(rng.choice([8, 16, 32, 64, 128]))
    B = int(rng.choice([1, 4, 16, 32]))
    e = int(rng.choice([1, 2, 4]))
    if (B * d * e) % 16:
        e = 2 if (B * d * 2) % 16 == 0 else 4
    if (B * d * e) % 16:
        B = 16
    L = int(rng.integers(1, 4))
    n_gpus = int(rng.choice([2, 4, 8, 16]))
    degrees = [p for p in (1, 2, 4, 8, 16) if p <= n_gpus and (p <= H and H % p == 0 or p > H and p % H == 0)]
    spec = []
    for _ in range(int(rng.integers(1, 12))):
        p0 = int(rng.choice(degrees))
        p1 = int(rng.choice(degrees))
        g0 = int(rng.integers(0, n_gpus // p0)) * p0
        g1 = int(rng.integers(0, n_gpus // p1)) * p1
        T = int(rng.choice([0, 1, int(rng.integers(2, 3 * B + 2)), int(rng.integers(40, 700))]))
        srid = [int(x) for x in rng.permutation(p0)] if p0 > 1 and rng.random() < 0.3 else None
        drid = [int(x) for x in rng.permutation(p1)] if p1 > 1 and rng.random() < 0.3 else None
        spec.append((T, (g0, p0), (g1, p1), srid, drid))
    mode = str(rng.choice(["one", "one", "per_gpu", "a2a", "ranges", "switch"]))
    cuts = sorted(set(int(x) for x in rng.integers(1, n_gpus, size=int(rng.integers(0, 4)))))
    ranges = list(zip([0] + cuts, cuts + [n_gpus]))
    return (L, H, d, B, e), n_gpus, spec, mode, int(rng.integers(0, 2)), ranges


@pytest.mark.parametrize("seed", range(SEED0, SEED0 + N_CASES))
def test_fuzz_parity(seed):
    geo, n_gpus, spec, mode, work_order, ranges = _case(seed)
    B = geo[3]
    nb = 2 * sum(-(-x[0] // B) for x in spec) + 64   # room for every source and destination on any pool
    run_parity(geo, [nb] * n_gpus, spec, seed=seed, per_gpu_launch=mode == "per_gpu", a2a=mode == "a2a",
               work_order=work_order, degrees=(2, 4, 8, 16), ranges=ranges if mode == "ranges" else None,
               one_call=mode == "switch")


N_WAVE_CASES = int(os.environ.get("FLYKV_FUZZ_WAVE_CASES", "12"))


@pytest.mark.parametrize("seed", range(SEED0, SEED0 + N_WAVE_CASES))
def test_fuzz_memory_bounded_waves(seed):
    """Random switches into pools too small for one shot, through the
    one-call kv_switch_waves (request-granular waves, or block-aligned token
    pieces, R20); the returned schedule replayed on the oracle wave by wave
    (its own source-table slicing, its own allocator): every wave's tables,
    then the whole pools and allocator state, bit-exact.  A switch that does
    not fit even piecewise must fail with no state change."""
    import torch

    import synth
    from helpers import oracle_alloc
    from oracle import oracle as O
    from paper_2602_22593_b200 import flykv as F
    from paper_2602_22593_b200.engine import KVSwitchEngine
    rng = np.random.default_rng(70000 + seed)
    H = int(rng.choice([1, 2, 4, 8]))
    geo = (int(rng.integers(1, 3)), H, int(rng.choice([32, 64, 128])), 16, 2)
    og = O.Geom(*geo)
    n_gpus = 8
    degrees = [p for p in (1, 2, 4, 8) if (p <= H and H % p == 0) or (p > H and p % H == 0)]
    spec = []
    for _ in range(int(rng.integers(2, 10))):
        p0, p1 = int(rng.choice(degrees)), int(rng.choice(degrees))
        spec.append((int(rng.integers(1, 1500)), (int(rng.integers(0, n_gpus // p0)) * p0, p0),
                     (int(rng.integers(0, n_gpus // p1)) * p1, p1)))
    need = [0] * n_gpus
    for T, s, d in spec:
        for g in range(s[0], s[0] + s[1]):
            need[g] += O.num_blocks(og, T, s[1])
    nb = [int(max(need) * rng.uniform(1.05, 1.6)) + 8] * n_gpus
    eng = KVSwitchEngine(F.geometry(*geo), nb, "cuda:0")
    for g, t in enumerate(eng.pools.tensors):
        synth.fill_hash_torch(t, g, seed=seed + 3)
    held = [np.zeros(n, dtype=np.uint8) for n in nb]
    reqs = []
    for i, (T, s, d) in enumerate(spec):
        reqs.append((i, T, s, oracle_alloc(eng.cache, held, s, O.num_blocks(og, T, s[1])), d))
    M = O.block_bytes(og)
    for (_, T, s, ids, d) in reqs:     # replicated sources identical (R10)
        if s[1] > H:
            rep = s[1] // H
            idx = torch.as_tensor(np.asarray(ids, dtype=np.int64), device="cuda:0")
            for r in range(s[1]):
                if r % rep:
                    eng.pools.tensors[s[0] + r][:, idx] = eng.pools.tensors[s[0] + r - r % rep][:, idx]
    torch.cuda.synchronize()
    host = [t.cpu().numpy().reshape(-1).copy() for t in eng.pools.tensors]
    split = bool(rng.integers(0, 2))
    masks = [eng.cache.held_mask(g).copy() for g in range(n_gpus)]
    try:
        waves, plans = F.kv_switch_waves(eng.cache, reqs, split=split, stream=eng.stream)
    except F.FlyKVError as e:   # does not fit even piecewise: nothing may have changed
        assert e.name == "KV_ERR_OUT_OF_BLOCKS" and not e.plans
        assert all(np.array_equal(eng.cache.held_mask(g), masks[g]) for g in range(n_gpus))
        return
    torch.cuda.synchronize()
    for wave, plan in zip(waves, plans):
        pieces = []
        for i, t0, t1 in wave:
            _, T, s, ids, d = reqs[i]
            b0 = O.block_tokens(og, s[1])
            pieces.append(O.Req(t1 - t0, s, list(ids[t0 // b0: -(-t1 // b0)]), d))
        st, otabs = O.switch(og, host, held, pieces)
        assert st == 0
        assert [list(a) for a in plan.dst_tables()] == [list(b) for b in otabs]
    for g in range(n_gpus):
        assert np.array_equal(eng.cache.held_mask(g), held[g])
        assert np.array_equal(eng.pools.tensors[g].cpu().numpy().reshape(-1), host[g]), f"pool {g}"
