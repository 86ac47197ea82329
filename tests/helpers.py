"""Test helpers.  Block IDs handed to the oracle never come from the product:
oracle_alloc computes the expected IDs with the brute-force oracle's own
allocator (lowest IDs free on every GPU of the group, R6/R8), checks that the
product's kv_alloc chose the same ones, and returns the oracle's list."""
import numpy as np

from oracle import brute


def oracle_alloc(cache, held, group, n):
    """held: oracle-side per-GPU uint8 masks (updated).  Returns int32 IDs."""
    want = brute.lowest_common_free(held, group, n)
    got = cache.alloc(group, n)
    assert want is not None and [int(x) for x in got] == want, (group, n, list(got)[:8], (want or [])[:8])
    for r in range(group[1]):
        held[group[0] + r][want] = 1
    return np.asarray(want, dtype=np.int32)
