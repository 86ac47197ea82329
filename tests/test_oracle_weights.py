"""Pins for the weight-view oracle (Eq.1), CPU only."""
import numpy as np
import pytest

from oracle import weights as W


def test_spec_examples():
    """O rows=8 (the sharded input extent), m=4, r=0 -> offset 0, extent 2;
    m=3 on extent 8 -> IndivisibleExtent; QKV with 24 output features, m=2,
    r=1 -> 12 features."""
    Wo = np.arange(5 * 8, dtype=np.float64).reshape(5, 8)  # [out=5, in=8]
    (v,) = W.view_row(Wo, 0, 4)
    assert v.shape == (5, 2) and np.shares_memory(v, Wo) and v[0, 0] == Wo[0, 0]
    with pytest.raises(W.IndivisibleExtent):
        W.view_row(Wo, 0, 3)
    with pytest.raises(W.RankOutOfRange):
        W.view_row(Wo, 4, 4)
    Wqkv = np.zeros((24, 8))  # Hq = Hkv = 2, d = 4
    segs = W.view_qkv(Wqkv, 1, 2, 2, 2, 4)
    assert sum(s.shape[0] for s in segs) == 12


@pytest.mark.parametrize("m", [1, 2, 4, 8])
@pytest.mark.parametrize("Hq,Hkv", [(8, 8), (8, 2), (16, 4), (8, 1)])
def test_qkv_views_tile_and_align(m, Hq, Hkv):
    """Views are zero-copy (share memory), head-aligned; Q slices tile
    the Q extent; K/V heads are disjoint when m <= Hkv and replicated
    m/Hkv times otherwise (GQA, R2)."""
    d, hidden = 4, 6
    Wf = np.random.default_rng(0).standard_normal(((Hq + 2 * Hkv) * d, hidden))
    qrows, krows = [], []
    for r in range(m):
        segs = W.view_qkv(Wf, r, m, Hq, Hkv, d)
        assert all(np.shares_memory(s, Wf) for s in segs)
        assert all(s.shape[0] % d == 0 for s in segs)
        qrows.append(segs[0])
        krows.append(segs[1])
    assert np.array_equal(np.concatenate(qrows), Wf[:Hq * d])
    if m <= Hkv:
        assert np.array_equal(np.concatenate(krows), Wf[Hq * d:(Hq + Hkv) * d])
    else:
        rep = m // Hkv
        for r in range(m):
            h = r // rep
            assert np.array_equal(krows[r], Wf[(Hq + h) * d:(Hq + h + 1) * d])


@pytest.mark.parametrize("m", [1, 2, 4])
def test_toy_tp_forward_matches_dense(m):
    """Column-parallel then row-parallel with a final sum == dense, fp64."""
    rng = np.random.default_rng(7)
    x = rng.standard_normal((4, 16))
    W1 = rng.standard_normal((32, 16))
    W2 = rng.standard_normal((16, 32))
    dense = (x @ W1.T) @ W2.T
    assert np.max(np.abs(W.tp_forward_toy(x, W1, W2, m) - dense)) <= 1e-9
