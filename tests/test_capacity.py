"""Capacity arithmetic pinned to the paper's Table 2
(8xH200, Llama-3-70B: 264K / 959K / 2.3M / 1.9M tokens) and
SPEC's max_context examples."""
import pytest

from paper_2602_22593_b200 import capacity as cap

KV70 = cap.kv_bytes_per_token(80, 8, 128, 2)


def test_kv_bytes_per_token_examples():
    assert KV70 == 327_680
    assert cap.kv_bytes_per_token(32, 8, 128, 2) == 131_072
    assert cap.kv_bytes_per_token(1, 1, 1, 1) == 2


def test_spec_tiny_example():
    # S:243 ("tiny spec (kv=2 B/token, mem=1,000 B, weights=200 B, util=1.0) -> 800
    # tokens") is inconsistent with its own formula: 800 free bytes / 2 B per
    # token = 400 tokens.  The formula is what the pin follows.
    assert cap.max_context(1, 1000, 200, 2) == 400


def test_table2_linear_model():
    """Fitting C, W to the 4DPx2TP and 2DPx4TP rows predicts the 1DPx8TP row
    (2.3M) and recovers the bf16 weight size of Llama-3-70B
    (70.6e9 params x 2 B = 141.1 GB) -- the paper's Table 2 is this model."""
    f = cap.fit_two_points(2, 264e3, 4, 959e3, KV70)
    assert f.weight_bytes == pytest.approx(141.1e9, rel=0.01)
    p8 = cap.max_context(8, f.per_gpu_bytes, f.weight_bytes, KV70)
    assert p8 == pytest.approx(2.3e6, rel=0.03)
    # the dynamic 1.9M row corresponds to a per-GPU reserve for
    # reconfiguration support of ~18 GB, "within 17%" of static TP8
    reserve = f.per_gpu_bytes - (1.9e6 * KV70 + f.weight_bytes) / 8
    assert 10e9 < reserve < 25e9
    assert cap.max_context(8, f.per_gpu_bytes, f.weight_bytes, KV70, reserve_bytes=reserve) == pytest.approx(1.9e6,
                                                                                                            rel=0.01)


def test_monotone_in_degree():
    f = cap.fit_two_points(2, 264e3, 4, 959e3, KV70)
    vals = [cap.max_context(p, f.per_gpu_bytes, f.weight_bytes, KV70) for p in (1, 2, 4, 8)]
    assert vals == sorted(vals) and vals[0] == 0  # one H200 cannot hold the weights + any KV


def test_relayout_reserve():
    # 128K-token Llama-3.1-8B request promoted to TP8: ceil(131072/128) blocks x 64 KiB x 32 layers per rank
    assert cap.relayout_reserve_bytes(131072, 32, 8, 128, 16, 4, 8) == 1024 * 65536 * 32


def test_table2_at_b200_memory():
    """The B200 table (capacity.table2 with the box's measured total memory,
    profiles/r02_n4_pool_capacity.json): the H200 model rows reproduce the
    paper's Table 2, KV bytes per token come from kv_layout, and
    the B200 rows scale by the memory ratio (weights unchanged)."""
    t = cap.table2(191502876672)
    assert t["kv_bytes_per_token"] == KV70
    model = [r["model_h200_tokens"] for r in t["rows"]]
    assert model[0] == 264000 and model[1] == 959000
    assert model[2] == pytest.approx(2.3e6, rel=0.03) and model[3] == pytest.approx(1.9e6, rel=1e-3)
    b200 = [r["tokens"] for r in t["rows"]]
    assert b200 == sorted(b200[:3]) + [b200[3]] and all(x % 16 == 0 for x in b200)
    assert b200[2] > b200[3] > b200[1]          # dynamic sits between static TP4 and TP8, as on H200
    # per-GPU bytes scale with total memory at the fitted utilisation
    assert t["per_gpu_bytes"] == pytest.approx(t["utilisation_of_total"] * 191502876672)
