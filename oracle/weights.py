"""Oracle for the Model Weights Manager's zero-copy shard view (Eq.1).

ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header).

    W_active^(r) = View(W_full, dim, r, m)                         (Eq.1)

Weights are stored PyTorch-style as [out, in] (rows = output features).
 * column-parallel (the fused W^QKV, also Up/Gate): rank r takes a
   slice of the OUTPUT features = a row range of the [out, in] storage;
   for the fused QKV (stacked [Q; K; V], R17) the slice is head-aligned:
   Q heads [r*Hq/m, (r+1)*Hq/m), and K/V heads [r*Hkv/m, ...) when m <= Hkv,
   else the single replicated KV head r // (m/Hkv) (GQA, R2);
 * row-parallel (W^O, Down): rank r takes a slice of the INPUT
   features = a column range [r*in/m, (r+1)*in/m) of the storage.
Each view is returned as numpy *views* of the full array (no copy).
"""
from __future__ import annotations

import numpy as np


class RankOutOfRange(ValueError):
    pass


class IndivisibleExtent(ValueError):
    pass


def _check(r, m, extent):
    if m < 1 or r < 0 or r >= m:
        raise RankOutOfRange((r, m))
    if extent % m:
        raise IndivisibleExtent((extent, m))


def view_col(W: np.ndarray, r: int, m: int):
    out = W.shape[0]
    _check(r, m, out)
    k = out // m
    return [W[r * k:(r + 1) * k, :]]


def view_row(W: np.ndarray, r: int, m: int):
    inn = W.shape[1]
    _check(r, m, inn)
    k = inn // m
    return [W[:, r * k:(r + 1) * k]]


def view_qkv(W: np.ndarray, r: int, m: int, Hq: int, Hkv: int, d: int):
    assert W.shape[0] == (Hq + 2 * Hkv) * d
    _check(r, m, Hq)
    q = Hq // m
    segs = [W[r * q * d:(r + 1) * q * d, :]]
    if m <= Hkv:
        _check(r, m, Hkv)
        k = Hkv // m
        h0, nh = r * k, k
    else:
        if m % Hkv:
            raise IndivisibleExtent((m, Hkv))
        h0, nh = r // (m // Hkv), 1
    kbase = Hq * d
    vbase = (Hq + Hkv) * d
    segs.append(W[kbase + h0 * d:kbase + (h0 + nh) * d, :])
    segs.append(W[vbase + h0 * d:vbase + (h0 + nh) * d, :])
    return segs


def tp_forward_toy(x, W1, W2, m):
    """Megatron MLP-style pair: column-parallel W1 then row-parallel W2, the
    partial outputs summed (the all-reduce).  fp64."""
    y = np.zeros((x.shape[0], W2.shape[0]), dtype=np.float64)
    for r in range(m):
        (w1,) = view_col(W1, r, m)
        (w2,) = view_row(W2, r, m)
        y += (x @ w1.T) @ w2.T
    return y
