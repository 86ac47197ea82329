"""Oracle for the consumer proof: single-query attention.

ORACLE -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.py header).

    out = softmax(scale * K q) V        (plain definition, fp64)

K, V: [T, d] (the logical KV of one head of one request, as located by
oracle.locate), q: [d].  Pinned in tests/test_oracle_attention.py.
"""
import numpy as np


def decode_attention(K, V, q, scale):
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    s = K @ np.asarray(q, dtype=np.float64) * float(scale)
    p = np.exp(s - s.max())
    return (p / p.sum()) @ V
