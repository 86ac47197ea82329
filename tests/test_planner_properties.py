"""Property tests of the host allocator/planner (hypothesis, CPU only, fake
pool pointers): random sequences of reserve/alloc/free/plan/commit/destroy
keep the paper's invariants -- conservation allocated + free == num_blocks
per GPU, uniform IDs across a TP group (R6), transactional failures
(S:207), byte invariance of what the plan moves (also per sender, over the
kernels' work order), and agreement with the oracle's allocator."""
import numpy as np
import pytest

hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

from helpers import oracle_alloc  # noqa: E402
from oracle import brute  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2602_22593_b200 import flykv as F  # noqa: E402

N_GPUS = 8


def _cache(H, nb):
    g = F.geometry(2, H, 8, 4, 2)
    bases = [[(1 << 40) + (r << 36) + (l << 30) for l in range(2)] for r in range(N_GPUS)]
    return F.KVCache(g, [nb] * N_GPUS, bases, (2, 4, 8))


group_st = st.sampled_from([1, 2, 4, 8]).flatmap(
    lambda p: st.tuples(st.integers(0, N_GPUS // p - 1).map(lambda k: k * p), st.just(p)))


@settings(max_examples=60, deadline=None, suppress_health_check=[HealthCheck.too_slow])
@given(H=st.sampled_from([1, 2, 4, 8]), nb=st.integers(8, 160),
       ops=st.lists(st.tuples(st.integers(0, 3), st.integers(0, 120), group_st, group_st), min_size=1, max_size=25))
def test_random_sequences_keep_invariants(H, nb, ops):
    c = _cache(H, nb)
    og = O.Geom(2, H, 8, 4, 2)
    held = [np.zeros(nb, dtype=np.uint8) for _ in range(N_GPUS)]  # oracle-side mirror
    live = []   # (rid, T, group, ids)
    rid = 0
    for kind, T, g1, g2 in ops:
        before = [c.held_mask(x).copy() for x in range(N_GPUS)]
        if kind == 0:  # admit a request (oracle-chosen IDs, checked against kv_alloc)
            n = O.num_blocks(og, T, g1[1])
            if brute.lowest_common_free(held, g1, n) is None:
                with pytest.raises(F.FlyKVError) as e:
                    c.alloc(g1, n)
                assert e.value.name == "KV_ERR_OUT_OF_BLOCKS"
                assert all(np.array_equal(c.held_mask(x), before[x]) for x in range(N_GPUS))
                continue
            ids = oracle_alloc(c, held, g1, n)
            live.append((rid, T, g1, ids))
            rid += 1
        elif kind == 1 and live:  # finish a request
            r_, T_, g_, ids_ = live.pop(T % len(live))
            c.free(g_, ids_)
            for r in range(g_[1]):
                held[g_[0] + r][ids_] = 0
        elif kind in (2, 3) and live:  # switch some requests to g2 (commit) or abandon the plan
            k = 1 + T % len(live)
            moving = live[:k]
            reqs = [(r_, T_, g_, ids_, g2) for (r_, T_, g_, ids_) in moving]
            try:
                plan = c.plan_switch(reqs)
            except F.FlyKVError as e:
                assert e.name == "KV_ERR_OUT_OF_BLOCKS"
                assert all(np.array_equal(c.held_mask(x), before[x]) for x in range(N_GPUS))
                continue
            ost, otabs = O.switch(og, None, [h.copy() for h in held],
                                  [O.Req(T_, g_, list(ids_), g2) for (_, T_, g_, ids_) in moving], copy=False)
            assert ost == 0
            tabs = plan.dst_tables()
            assert [list(a) for a in tabs] == [list(b) for b in otabs]
            stt, mat = plan.stats()
            want = sum(2 * 2 * H * (-(-T_ // 4)) * 4 * 8 * 2 * O.replicas(og, g2[1])
                       for (_, T_, g_, _) in moving if tuple(g_) != tuple(g2))
            assert stt["payload_bytes"] == want == int(mat.sum())
            # the kernels' work order covers exactly the plan's bytes, sender by sender
            for x in range(N_GPUS):
                rows = plan.work_order(x)
                assert np.array_equal(rows[:, :N_GPUS].sum(0), mat[x])
            assert stt["n_atom_slots"] >= stt["n_atoms"]
            if kind == 2:
                plan.commit()
                O.switch(og, None, held, [O.Req(T_, g_, list(ids_), g2) for (_, T_, g_, ids_) in moving],
                         copy=False)
                live = [(r_, T_, g2, t) for (r_, T_, _, _), t in zip(moving, tabs)] + live[k:]
            else:
                plan.destroy()
                assert all(np.array_equal(c.held_mask(x), before[x]) for x in range(N_GPUS))
        # invariants after every op
        for x in range(N_GPUS):
            assert np.array_equal(c.held_mask(x), held[x])
            assert c.free_count(x) + int(held[x].sum()) == nb
        for (_, T_, g_, ids_) in live:  # uniform IDs across each group (R6)
            for r in range(g_[1]):
                assert held[g_[0] + r][ids_].all()
