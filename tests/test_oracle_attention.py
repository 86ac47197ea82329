"""Pins of oracle/attention.py against closed forms."""
import numpy as np

from oracle.attention import decode_attention


def test_uniform_scores_average_values():
    """Equal scores -> the arithmetic mean of V (softmax of a constant)."""
    rng = np.random.default_rng(0)
    V = rng.standard_normal((7, 16))
    K = np.ones((7, 16))
    assert np.allclose(decode_attention(K, V, np.ones(16), 0.1), V.mean(0), atol=1e-12)


def test_dominant_key_selects_its_value():
    """One key aligned with q at a huge scale -> that row of V."""
    rng = np.random.default_rng(1)
    V = rng.standard_normal((5, 8))
    K = np.zeros((5, 8))
    K[3] = 1.0
    assert np.allclose(decode_attention(K, V, np.ones(8), 1e3), V[3], atol=1e-12)


def test_two_keys_closed_form():
    """Two keys: weights are the logistic of the score difference."""
    V = np.array([[1.0, 0.0], [0.0, 1.0]])
    K = np.array([[1.0, 0.0], [0.0, 1.0]])
    q = np.array([2.0, 0.5])
    w0 = 1.0 / (1.0 + np.exp(-(2.0 - 0.5)))
    assert np.allclose(decode_attention(K, V, q, 1.0), [w0, 1 - w0], atol=1e-12)
