"""KV capacity arithmetic (Table 2 of the paper).

Maximum context a TP-p instance can hold, once the weights (sharded p ways,
P:273-284) are resident:

    max_context(p) = floor( (p * C - W) / kv_bytes_per_token )   (floored to B(p))

C = bytes per GPU available to weights + KV, W = total weight bytes,
kv_bytes_per_token = 2 * L * H_kv * d * e (K and V of every layer, R1).
This is the same linear model the paper's Table 2 follows: fitting C and W to
two of its static rows reproduces the third and recovers Llama-3-70B's bf16
weight size (tests/test_capacity.py).  Host-side planning only.
"""
from __future__ import annotations

from dataclasses import dataclass


def kv_bytes_per_token(L: int, H: int, d: int, e: int = 2) -> int:
    return 2 * L * H * d * e


def max_context(p: int, per_gpu_bytes: float, weight_bytes: float, kv_per_token: int, block_tokens: int = 1,
                reserve_bytes: float = 0.0) -> int:
    free = p * (per_gpu_bytes - reserve_bytes) - weight_bytes
    if free <= 0:
        return 0
    t = int(free // kv_per_token)
    return t - t % max(1, block_tokens)


@dataclass
class Fit:
    per_gpu_bytes: float
    weight_bytes: float


def fit_two_points(p1: int, t1: float, p2: int, t2: float, kv_per_token: int) -> Fit:
    """Solve p*C - W = t*kv for (C, W) from two (degree, max context) rows."""
    c = (t2 - t1) * kv_per_token / (p2 - p1)
    w = p1 * c - t1 * kv_per_token
    return Fit(c, w)


def relayout_reserve_bytes(T: int, L: int, H: int, d: int, B: int, p_src: int, p_dst: int, e: int = 2) -> float:
    """Per-GPU destination bytes a live re-layout of one T-token request
    needs next to its sources (R13): ceil(T / B(p_dst)) blocks of M bytes per
    layer on each destination rank -- block count and M from the library's
    kv_blocks_for / kv_layout (Eq.2, Eq.3, M_block).  With memory-bounded
    waves (kv_plan_waves) this bounds the transient reserve of a promotion."""
    from . import flykv
    g = flykv.geometry(L, H, d, B, e)
    _, _, M = flykv.kv_layout(g, p_dst)
    return flykv.kv_blocks_for(g, T, p_dst) * M * L


H200_TOTAL_BYTES = 141e9   # the paper's GPU, 141 GB HBM3e (public spec)
TABLE2_ROWS = (("Static 4DPx2TP", 2, 264e3), ("Static 2DPx4TP", 4, 959e3), ("Static 1DPx8TP", 8, 2.3e6))
TABLE2_DYNAMIC = 1.9e6


def table2(total_bytes: float, L: int = 80, H: int = 8, d: int = 128, B: int = 16, e: int = 2) -> dict:
    """Table 2 at another GPU's memory: fit the linear model to the
    paper's two lower static rows (H200), keep its weight size and its
    utilisation fraction of total memory, rescale per-GPU bytes to
    total_bytes, and keep the dynamic row's fitted per-GPU reserve.  KV bytes
    per token from the library (kv_layout: M_block eq., Eq.2).  Defaults:
    Llama-3-70B.  Returns the fit and one row per configuration."""
    from . import flykv
    g = flykv.geometry(L, H, d, B, e)
    _, bt, M = flykv.kv_layout(g, 1)
    kv_tok = M * L // bt
    fit = fit_two_points(TABLE2_ROWS[0][1], TABLE2_ROWS[0][2], TABLE2_ROWS[1][1], TABLE2_ROWS[1][2], kv_tok)
    util = fit.per_gpu_bytes / H200_TOTAL_BYTES
    C = util * total_bytes
    reserve = fit.per_gpu_bytes - (TABLE2_DYNAMIC * kv_tok + fit.weight_bytes) / 8
    rows = []
    for name, p, paper in TABLE2_ROWS:
        rows.append({"config": name, "gpus_per_instance": p, "paper_h200_tokens": paper,
                     "model_h200_tokens": max_context(p, fit.per_gpu_bytes, fit.weight_bytes, kv_tok),
                     "tokens": max_context(p, C, fit.weight_bytes, kv_tok, block_tokens=bt)})
    rows.append({"config": "Flying Serving (dynamic, up to 8 GPUs)", "gpus_per_instance": "dynamic",
                 "paper_h200_tokens": TABLE2_DYNAMIC,
                 "model_h200_tokens": max_context(8, fit.per_gpu_bytes, fit.weight_bytes, kv_tok, reserve_bytes=reserve),
                 "tokens": max_context(8, C, fit.weight_bytes, kv_tok, reserve_bytes=reserve, block_tokens=bt)})
    return {"kv_bytes_per_token": kv_tok, "total_bytes": total_bytes, "fit_per_gpu_bytes_h200": fit.per_gpu_bytes,
            "fit_weight_bytes": fit.weight_bytes, "utilisation_of_total": util, "per_gpu_bytes": C,
            "dynamic_reserve_bytes_per_gpu": reserve, "rows": rows}
