"""Serving soak: a long random sequence of admissions, completions and live
DP<->TP switches (merges, splits, promotions, rank-ID re-assignments, waves)
on 8 virtual ranks.  Every request carries its own content pattern written at
admission; after hundreds of switches every live request's KV, read through
the oracle's atom map of its *current* layout, must still equal that pattern,
and the allocator must conserve blocks and match the oracle's
allocator state step by step."""
import os

import numpy as np
import pytest

import synth
from helpers import oracle_alloc
from oracle import brute
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GEO = (2, 8, 64, 16, 2)
N_GPUS = 8
NB = 1500


def _atoms(og, nb, req):
    """(gpu, word offset, logical atom index) of every stored atom copy of
    req's current layout: atom_map enumerates (l, kv, h, c, replica j) with
    j innermost, so all replicas of one logical atom share its index."""
    T, grp, tab, rid = req["T"], req["grp"], req["tab"], req["rid"]
    _, _, dg, do = O.atom_map(og, nb, T, grp, tab, grp, tab, rid, rid)
    logical = np.arange(len(dg)) // O.replicas(og, grp[1])
    return dg.astype(np.int64), do // 4, logical


def _pattern(seed, logical, atom_words, dev):
    lg = torch.as_tensor(logical, device=dev)
    idx = lg[:, None] * atom_words + torch.arange(atom_words, dtype=torch.int64, device=dev)[None, :]
    return synth.hash32_torch(7, idx, seed=seed)


def _write(flat, g, w, vals, atom_words, ar):
    for gd in np.unique(g):
        m = torch.as_tensor(g == gd, device=vals.device)
        idx = torch.as_tensor(w, device=vals.device)[m][:, None] + ar[None, :]
        flat[int(gd)][idx] = vals[m]


def _read(flat, g, w, atom_words, ar, dev):
    out = torch.empty((len(g), atom_words), dtype=torch.int32, device=dev)
    for gd in np.unique(g):
        m = torch.as_tensor(g == gd, device=dev)
        idx = torch.as_tensor(w, device=dev)[m][:, None] + ar[None, :]
        out[m] = flat[int(gd)][idx]
    return out


SEEDS = [int(x) for x in os.environ.get("FLYKV_SOAK_SEEDS", "0,1,2").split(",")]
ITERS = int(os.environ.get("FLYKV_SOAK_ITERS", "1200"))


CASES = [(s, GEO) for s in SEEDS] + [(SEEDS[0], (2, 1, 64, 16, 2)), (SEEDS[0], (2, 2, 128, 16, 2))]


@pytest.mark.parametrize("seed,geo", CASES)
def test_serving_soak(seed, geo):
    """H_kv = 8 (no replication) on every seed; H_kv = 1 and 2 (GQA
    replication at TP > H_kv: the TMA replica kernel, replicated sources) on
    the first seed, in strict replica mode (R10) with every other switch
    through the one-call kv_switch, which verifies the replicas first."""
    F = pytest.importorskip("paper_2602_22593_b200.flykv")
    from paper_2602_22593_b200.engine import KVSwitchEngine
    rng = np.random.default_rng(seed)
    og = O.Geom(*geo)
    nb = [NB] * N_GPUS
    eng = KVSwitchEngine(F.geometry(*geo), nb, "cuda:0")
    strict = geo[1] < N_GPUS
    if strict:
        eng.cache.set_strict(True)
    dev = torch.device("cuda:0")
    flat = [t.reshape(-1).view(torch.int32) for t in eng.pools.tensors]
    atom_words = og.B * og.d * og.e // 4
    ar = torch.arange(atom_words, dtype=torch.int64, device=dev)
    held = [np.zeros(NB, dtype=np.uint8) for _ in range(N_GPUS)]  # oracle-side allocator mirror
    live = {}
    next_id = 0
    switches = 0

    def groups(p):
        return [(k * p, p) for k in range(N_GPUS // p)]

    for it in range(ITERS):
        op = rng.random()
        if op < 0.35 or not live:  # admit into a random layout
            p = int(rng.choice([1, 1, 2, 4, 8]))
            grp = groups(p)[int(rng.integers(len(groups(p))))]
            T = int(rng.integers(1, 600))
            rid = [int(x) for x in rng.permutation(p)] if rng.random() < 0.3 else None
            n = O.num_blocks(og, T, p)
            if brute.lowest_common_free(held, grp, n) is None:
                with pytest.raises(F.FlyKVError):
                    eng.cache.alloc(grp, n)
                continue
            tab = oracle_alloc(eng.cache, held, grp, n)
            req = {"T": T, "grp": grp, "tab": tab, "rid": rid, "seed": 1000 * seed + next_id}
            g, w, lg = _atoms(og, nb, req)
            _write(flat, g, w, _pattern(req["seed"], lg, atom_words, dev), atom_words, ar)
            live[next_id] = req
            next_id += 1
        elif op < 0.5:  # complete a request
            k = int(rng.choice(list(live)))
            req = live.pop(k)
            eng.cache.free(req["grp"], req["tab"])
            for r in range(req["grp"][1]):
                held[req["grp"][0] + r][req["tab"]] = 0
        else:  # switch a random subset to one destination layout
            p = int(rng.choice([1, 2, 4, 8]))
            dst = groups(p)[int(rng.integers(len(groups(p))))]
            keys = [k for k in live if rng.random() < 0.4][:12]
            if not keys:
                continue
            drid = [int(x) for x in rng.permutation(p)] if rng.random() < 0.3 else None
            reqs = [(k, live[k]["T"], live[k]["grp"], live[k]["tab"], dst, live[k]["rid"], drid) for k in keys]
            oreqs = [O.Req(live[k]["T"], live[k]["grp"], list(live[k]["tab"]), dst, live[k]["rid"], drid)
                     for k in keys]
            try:
                waves = F.kv_plan_waves(eng.cache, reqs)
            except F.FlyKVError as e:
                assert e.name == "KV_ERR_OUT_OF_BLOCKS"
                continue
            for a, b in waves:
                if strict and switches % 2:   # strict mode: kv_switch verifies replicated sources first
                    plan = F.kv_switch(eng.cache, reqs[a:b], eng.stream)
                else:
                    plan, tables, _ = eng.switch(reqs[a:b], read_back=True)
                st, otabs = O.switch(og, None, held, oreqs[a:b], copy=False)
                assert st == 0
                assert [list(x) for x in plan.dst_tables()] == [list(y) for y in otabs]
                for k, t in zip(keys[a:b], plan.dst_tables()):
                    live[k].update(grp=dst, tab=t, rid=drid)
                switches += 1
        for gpu in range(N_GPUS):
            assert eng.cache.free_count(gpu) + int(held[gpu].sum()) == NB
        if it % 100 == 99:
            torch.cuda.synchronize()
            for g_ in range(N_GPUS):
                assert np.array_equal(eng.cache.held_mask(g_), held[g_])
    torch.cuda.synchronize()
    assert switches > ITERS // 6
    for k, req in live.items():
        g, w, lg = _atoms(og, nb, req)
        got = _read(flat, g, w, atom_words, ar, dev)
        assert torch.equal(got, _pattern(req["seed"], lg, atom_words, dev)), f"request {k} corrupted"
