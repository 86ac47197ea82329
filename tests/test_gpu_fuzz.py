"""Randomised parity fuzz (GPU): random geometry (layers, KV heads, head_dim,
block size, element size), 2-16 virtual pools, random merges / splits /
lateral moves / no-ops with random rank-ID permutations on both sides
(incl. replicated sources and GQA destinations), random lengths incl. 0 and
tails, either kernel work order, and one of the launch paths (one launch,
per-pool launches, kv_reshard_range over a random partition of the pools,
the one-call kv_switch, pack -> all-to-all -> unpack); whole pools, tables and
allocator state bit-exact against the oracle (run_parity).  FLYKV_FUZZ_CASES
(default 24) sets the count; FLYKV_FUZZ_SEED0 the first seed."""
import os

import numpy as np
import pytest

from test_gpu_parity import run_parity

pytestmark = pytest.mark.gpu

N_CASES = int(os.environ.get("FLYKV_FUZZ_CASES", "24"))
SEED0 = int(os.environ.get("FLYKV_FUZZ_SEED0", "0"))


def _case(seed):
    rng = np.random.default_rng(50000 + seed)
    H = int(rng.choice([1, 2, 4, 8, 16]))
    d = int(rng.choice([8, 16, 32, 64, 128]))
    B = int(rng.choice([1, 4, 16, 32]))
    e = int(rng.choice([1, 2, 4]))
    if (B * d * e) % 16:
        e = 2 if (B * d * 2) % 16 == 0 else 4
    if (B * d * e) % 16:
        B = 16
    L = int(rng.integers(1, 4))
    n_gpus = int(rng.choice([2, 4, 8, 16]))
    degrees = [p for p in (1, 2, 4, 8, 16) if p <= n_gpus and (p <= H and H % p == 0 or p > H and p % H == 0)]
    spec = []
    for _ in range(int(rng.integers(1, 12))):
        p0 = int(rng.choice(degrees))
        p1 = int(rng.choice(degrees))
        g0 = int(rng.integers(0, n_gpus // p0)) * p0
        g1 = int(rng.integers(0, n_gpus // p1)) * p1
        T = int(rng.choice([0, 1, int(rng.integers(2, 3 * B + 2)), int(rng.integers(40, 700))]))
        srid = [int(x) for x in rng.permutation(p0)] if p0 > 1 and rng.random() < 0.3 else None
        drid = [int(x) for x in rng.permutation(p1)] if p1 > 1 and rng.random() < 0.3 else None
        spec.append((T, (g0, p0), (g1, p1), srid, drid))
    mode = str(rng.choice(["one", "one", "per_gpu", "a2a", "ranges", "switch"]))
    cuts = sorted(set(int(x) for x in rng.integers(1, n_gpus, size=int(rng.integers(0, 4)))))
    ranges = list(zip([0] + cuts, cuts + [n_gpus]))
    return (L, H, d, B, e), n_gpus, spec, mode, int(rng.integers(0, 2)), ranges


@pytest.mark.parametrize("seed", range(SEED0, SEED0 + N_CASES))
def test_fuzz_parity(seed):
    geo, n_gpus, spec, mode, work_order, ranges = _case(seed)
    B = geo[3]
    nb = 2 * sum(-(-x[0] // B) for x in spec) + 64   # room for every source and destination on any pool
    run_parity(geo, [nb] * n_gpus, spec, seed=seed, per_gpu_launch=mode == "per_gpu", a2a=mode == "a2a",
               work_order=work_order, degrees=(2, 4, 8, 16), ranges=ranges if mode == "ranges" else None,
               one_call=mode == "switch")
