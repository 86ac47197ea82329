"""Kernel work order (kv_cache_set_work_order) and the ordered
link model of bench.py, on CPU (fake pool pointers, nothing is moved).

The order decides only WHEN each (atom, replica) is written, never where:
the byte accounting of every order must equal the plan's byte matrix, and
the GPU parity tests (tests/test_gpu_parity.py) run with the default mixed
order.  Here: the per-range accounting of kv_plan_work_order sums to the
byte matrix for both orders on every degree pair; the mixed order keeps
each sender's destination mix constant over its ranges while plan order
visits receivers one after another; and the fluid link model reproduces
closed forms (a lone local copy is HBM-bound, a symmetric exchange is
link-bound, N senders into one receiver take N times one sender's time)."""
import numpy as np
import pytest

import bench
from paper_2602_22593_b200 import flykv as F


def fake_cache(geo, nb, degrees=(2, 4, 8)):
    g = F.geometry(*geo)
    bases = [[(1 << 40) + (gpu << 36) + (l << 30) for l in range(geo[0])] for gpu in range(len(nb))]
    return F.KVCache(g, nb, bases, degrees)


def _tp_to_dp(cache, n, T, seed=0):
    """Requests in TP-n on GPUs [0, n) split back to DP engines i mod n."""
    rng = np.random.default_rng(seed)
    reqs = []
    for i, t in enumerate(T):
        ids = cache.alloc((0, n), F.kv_blocks_for(cache.geom, t, n))
        reqs.append((i, t, (0, n), ids, (i % n, 1)))
    rng.shuffle(reqs)
    return reqs


@pytest.mark.parametrize("order", [0, 1])
@pytest.mark.parametrize("H,p0,p1", [(8, 1, 8), (8, 8, 1), (4, 2, 4), (2, 4, 1), (1, 1, 4), (4, 4, 2), (8, 2, 8)])
def test_work_order_rows_sum_to_byte_matrix(order, H, p0, p1):
    n = max(p0, p1)
    c = fake_cache((3, H, 64, 16, 2), [4096] * n)
    c.set_work_order(order)
    rng = np.random.default_rng(H * 100 + p0 * 10 + p1)
    reqs = []
    for i in range(24):
        T = int(rng.integers(1, 900))
        g0 = (i % (n // p0)) * p0
        ids = c.alloc((g0, p0), F.kv_blocks_for(c.geom, T, p0))
        g1 = ((i // 3) % (n // p1)) * p1
        reqs.append((i, T, (g0, p0), ids, (g1, p1)))
    plan = c.plan_switch(reqs)
    st, mat = plan.stats()
    reads = 0
    for g in range(n):
        rows = plan.work_order(g)
        assert rows.shape[1] == n + 1
        assert np.array_equal(rows[:, :n].sum(0), mat[g]), (g, rows[:, :n].sum(0), mat[g])
        reads += int(rows[:, n].sum())
    assert reads == st["n_atoms"] * st["atom_bytes"]
    assert st["n_atom_slots"] >= st["n_atoms"]
    plan.destroy()


def test_mixed_order_spreads_each_sender_over_its_receivers():
    """TP8 -> 8 x DP1: in plan order every range of a sender goes to one
    receiver and all senders start on the same one; in the mixed order every
    range carries the sender's whole-switch destination mix."""
    c = fake_cache((16, 8, 128, 16, 2), [8192] * 8)
    T = [512 + 97 * i for i in range(32)]
    reqs = _tp_to_dp(c, 8, T)
    c.set_work_order(0)
    p0 = c.plan_switch(reqs)
    first = [int(np.argmax(p0.work_order(g)[0, :8])) for g in range(8)]
    assert len(set(first)) == 1                      # all senders hit one receiver first
    r0 = p0.work_order(3)[:, :8]
    assert (r0 > 0).sum(1).mean() < 2.0               # plan order: about one receiver per range
    p0.destroy()
    c.set_work_order(1)
    p1 = c.plan_switch(reqs)
    _, mat = p1.stats()
    for g in range(8):
        rows = p1.work_order(g)[:-2, :8].astype(float)   # the last ranges hold the ragged ends of the buckets
        full = rows[rows.sum(1) > 0.9 * rows.sum(1).max()]
        assert len(full) > 0.9 * len(rows)
        mix = full / full.sum(1, keepdims=True)
        want = mat[g] / mat[g].sum()
        assert (full > 0).all()                       # every receiver in every range
        assert np.abs(mix - want).max() < 0.02        # constant mix (quantum granularity)
    p1.destroy()
    with pytest.raises(F.FlyKVError):
        c.set_work_order(7)


def test_link_model_closed_forms():
    hbm, link = 8000.0, 1000.0
    # a lone local copy: reads + writes of 8 GB on one GPU's HBM
    one = [np.array([[4e9, 4e9]])]
    assert bench.ordered_link_model(one, hbm, link) == pytest.approx(8e9 / 8e12)
    # symmetric exchange of 2 GB each way: link-bound
    ex = [np.array([[0, 2e9, 2e9]]), np.array([[2e9, 0, 2e9]])]
    assert bench.ordered_link_model(ex, hbm, link) == pytest.approx(2e9 / 1e12)
    # 4 senders (GPUs 1..4), 1 GB to each of the 4 other GPUs, in 4 pieces.
    n, b = 5, 1e9
    def piece(dst):
        r = np.zeros(n + 1)
        r[dst] = b
        r[n] = b
        return r
    # same visiting order on every sender (0, then the rest): receiver 0 is hit by all 4 at once first
    same = [np.zeros((0, n + 1))] + [np.array([piece(d) for d in [0] + [x for x in range(1, n) if x != s]])
                                     for s in range(1, n)]
    # rotated: at step k sender s targets a different receiver than every other sender
    rot = [np.zeros((0, n + 1))] + [np.array([piece((s + k) % n) for k in range(1, n)]) for s in range(1, n)]
    mix = [np.zeros((0, n + 1))] + [r.sum(0, keepdims=True) for r in rot[1:]]
    t_min = bench.nvlink_roofline(sum(np.pad(r[:, :n].sum(0, keepdims=True), ((s, n - 1 - s), (0, 0)))
                                      for s, r in enumerate(rot) if len(r)), hbm, link)[0]
    assert t_min == pytest.approx(4 * b / 1e12)                  # every sender's egress: 4 GB
    assert bench.ordered_link_model(rot, hbm, link) == pytest.approx(t_min)
    assert bench.ordered_link_model(mix, hbm, link) == pytest.approx(t_min)
    assert bench.ordered_link_model(same, hbm, link) > 1.5 * t_min   # the ingress hot-spot costs


def test_link_model_never_beats_t_min():
    """Any visiting order takes at least t_min: t_min is a
    lower bound, the ordered model a schedule.  Random byte rows, random
    orders, 2-8 GPUs; one row per GPU (perfect mixing) with no HBM limit in
    play reaches the link bound exactly when every sender is link-bound."""
    rng = np.random.default_rng(5)
    hbm, link = 8000.0, 800.0
    for trial in range(40):
        n = int(rng.integers(2, 9))
        pieces = []
        mat = np.zeros((n, n))
        for g in range(n):
            k = int(rng.integers(1, 6))
            rows = np.zeros((k, n + 1))
            for r in range(k):
                dests = rng.choice(n, size=int(rng.integers(1, n + 1)), replace=False)
                rows[r, dests] = rng.integers(1, 50, size=dests.size) * 1e8
                rows[r, n] = rows[r, :n].sum()
            pieces.append(rows)
            mat[g] = rows[:, :n].sum(0)
        t_min = bench.nvlink_roofline(mat, hbm, link)[0]
        t = bench.ordered_link_model(pieces, hbm, link)
        assert t >= t_min * (1 - 1e-9), (trial, t, t_min)
    # all-to-all of equal bytes, one mixed row per sender: exactly the egress bound
    n, b = 4, 1e9
    rows = [np.array([[b if d != g else 0.0 for d in range(n)] + [b * (n - 1)]]) for g in range(n)]
    mat = np.array([r[0, :n] for r in rows])
    assert bench.ordered_link_model(rows, hbm, link) == pytest.approx(bench.nvlink_roofline(mat, hbm, link)[0])
