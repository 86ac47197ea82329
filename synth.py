"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic (no block sizing, no head
ownership, no offsets): it only draws request lengths, places requests on
engines (the scheduler's choice, reading R11), shuffles block
IDs to fragment the pools, and fills pool bytes with a counter-based hash.
Both the oracle side and the CUDA side compute every layout quantity with
their own code and pass counts *into* these helpers.

Recipe:
  * lengths: uniform integers, numpy default_rng(seed=0), ranges from the
    paper's synthetic trace (prompts U[128,4000]) or BASELINE.json;
  * placement: round-robin by request index (R11);
  * source block IDs: per source group, a seeded permutation of the pool's
    block IDs (default_rng(seed=1)), consumed in request order -> scattered,
    fragmented tables;
  * contents: 32-bit word w of GPU g's pool = hash32(seed=2, g, w), the same
    counter hash on the device (torch int64 ops) and on the host (numpy).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------- workloads


@dataclass
class Workload:
    name: str
    L: int
    H: int
    d: int
    B: int
    e: int
    n_gpus: int
    T: list                      # tokens per request
    src: list                    # (first_gpu, degree) per request
    dst: list                    # (first_gpu, degree) per request
    tp_degrees: tuple = (2, 4, 8)
    note: str = ""
    extra: dict = field(default_factory=dict)

    def reversed(self) -> "Workload":
        return Workload(self.name + "-rev", self.L, self.H, self.d, self.B, self.e, self.n_gpus,
                        list(self.T), list(self.dst), list(self.src), self.tp_degrees, self.note)

    def tokens(self) -> int:
        return int(sum(self.T))


def lengths(n: int, lo: int, hi: int, seed: int = 0) -> list:
    rng = np.random.default_rng(seed)
    return [int(x) for x in rng.integers(lo, hi + 1, size=n)]


def tiny(n_req: int = 8, T: int = 256) -> Workload:
    """BASELINE configs[0]: 2 layers, 4 KV heads, d=64, B=16, 8 x 256 tokens,
    DP2 (request i on GPU i mod 2) -> TP2 {0,1}."""
    return Workload("tiny", 2, 4, 64, 16, 2, 2, [T] * n_req,
                    [(i % 2, 1) for i in range(n_req)], [(0, 2)] * n_req)


def llama8b_dp4_tp2x2(n_req: int = 64, seed: int = 0) -> Workload:
    """BASELINE configs[1]: Llama-3.1-8B-shaped cache (32 layers, 8 KV heads,
    d=128, B=16), 64 requests U{512..4096}, DP4 -> TP2x2 ({0,1},{2,3})."""
    T = lengths(n_req, 512, 4096, seed)
    src = [(i % 4, 1) for i in range(n_req)]
    dst = [((i % 4) // 2 * 2, 2) for i in range(n_req)]
    return Workload("llama3.1-8b DP4->TP2x2", 32, 8, 128, 16, 2, 4, T, src, dst)


def qwen32b_tp4x2_dp(n_req: int = 256, seed: int = 0) -> Workload:
    """BASELINE configs[2] (i): Qwen2.5-32B-shaped (64 layers, 8 KV heads),
    burst of 256 requests U{128..4000}, TP4x2 -> DP8."""
    T = lengths(n_req, 128, 4000, seed)
    src = [((i % 2) * 4, 4) for i in range(n_req)]
    dst = [((i % 2) * 4 + (i // 2) % 4, 1) for i in range(n_req)]
    return Workload("qwen2.5-32b TP4x2->DP8", 64, 8, 128, 16, 2, 8, T, src, dst)


def qwen32b_tp2x4_tp8(n_req: int = 256, seed: int = 0) -> Workload:
    """BASELINE configs[2] (ii): TP2x4 -> TP8."""
    T = lengths(n_req, 128, 4000, seed)
    src = [((i % 4) * 2, 2) for i in range(n_req)]
    dst = [(0, 8)] * n_req
    return Workload("qwen2.5-32b TP2x4->TP8", 64, 8, 128, 16, 2, 8, T, src, dst)


def llama70b_dp8_tp8(n_req: int = 64, seed: int = 0, H: int = 8) -> Workload:
    """BASELINE configs[3]: Llama-3-70B-shaped (80 layers, 8 KV heads),
    8 x DP1 -> TP8 (1 head/rank).  H=4 or H=1 gives the GQA-replication
    variants (TP8 > kv_heads)."""
    T = lengths(n_req, 512, 4096, seed)
    src = [(i % 8, 1) for i in range(n_req)]
    dst = [(0, 8)] * n_req
    return Workload(f"llama3-70b DP8->TP8 H{H}", 80, H, 128, 16, 2, 8, T, src, dst)


def weak_merge(n_gpus: int, per_engine: int = 8, engines_per_gpu: int = 2, seed: int = 0) -> Workload:
    """Weak-scaling series (round-1 review): Llama-3-70B geometry, two DP
    engines per GPU (so one GPU already has a real merge), 8 requests per
    engine with the same lengths T ~ U[512, 4096] on every engine, merged
    into TP groups of min(E, 8) engines (E = 2 x GPUs: TP2 on 1 GPU, TP4 on
    2, TP8 on 4, 2 x TP8 on 8).  Per-GPU bytes are the same at every N."""
    E = engines_per_gpu * n_gpus
    p = min(E, 8)
    Te = lengths(per_engine, 512, 4096, seed)
    T = [t for _ in range(E) for t in Te]
    src = [(e, 1) for e in range(E) for _ in range(per_engine)]
    dst = [((e // p) * p, p) for e in range(E) for _ in range(per_engine)]
    return Workload(f"llama3-70b weak DP{E}->TP{p}x{E // p} ({per_engine} req/engine, {engines_per_gpu} engines/GPU)",
                    80, 8, 128, 16, 2, E, T, src, dst)


def llama70b_fanout(n_req: int = 64, seed: int = 0) -> Workload:
    """BASELINE configs[3] (ii): single DP replica on GPU0 -> TP8 (the merge
    of a DP engine into one TP group).  Its sources sit at the
    top of GPU0's pool (src_top): uniform destination IDs (R6) then come from
    the low IDs every member has free, so GPUs 1-7 need pools only as large
    as their share of the destination -- the whole switch fits one B200."""
    T = lengths(n_req, 512, 4096, seed)
    return Workload("llama3-70b DP1(gpu0)->TP8", 80, 8, 128, 16, 2, 8, T,
                    [(0, 1)] * n_req, [(0, 8)] * n_req, extra={"src_top": True})


def long_context_tp4_tp8(n_short: int = 128, seed: int = 0, long_T: int = 131072) -> Workload:
    """BASELINE configs[4]: one 128K-token request in TP4{0-3} plus 128 short
    DP requests on GPUs 4-7, all promoted to TP8 (Llama-3.1-8B geometry)."""
    T = [long_T] + lengths(n_short, 128, 4000, seed)
    src = [(0, 4)] + [(4 + i % 4, 1) for i in range(n_short)]
    dst = [(0, 8)] * (n_short + 1)
    return Workload("long-context TP4+DP->TP8", 32, 8, 128, 16, 2, 8, T, src, dst)


def dp_to_tp(n_gpus: int, n_req: int, L=32, H=8, d=128, B=16, lo=512, hi=4096, seed=0) -> Workload:
    """DP_n -> TP_n merge of C2 geometry (used for the N-GPU bench sweep)."""
    T = lengths(n_req, lo, hi, seed)
    return Workload(f"DP{n_gpus}->TP{n_gpus}", L, H, d, B, 2, n_gpus, T,
                    [(i % n_gpus, 1) for i in range(n_req)], [(0, n_gpus)] * n_req)


def single_promotion(T: int = 4096) -> Workload:
    """One live 4K-token request promoted from a DP engine into TP8
    (Llama-3-70B geometry): the latency-bound end of the switch spectrum."""
    return Workload(f"llama3-70b single {T}-token DP1->TP8", 80, 8, 128, 16, 2, 8, [T], [(3, 1)], [(0, 8)])


WORKLOADS = {
    "tiny": tiny,
    "c2": llama8b_dp4_tp2x2,
    "c3i": qwen32b_tp4x2_dp,
    "c3ii": qwen32b_tp2x4_tp8,
    "c4": llama70b_dp8_tp8,
    "c4fan": llama70b_fanout,
    "c4gqa4": lambda **kw: llama70b_dp8_tp8(H=4, **kw),
    "c4gqa2": lambda **kw: llama70b_dp8_tp8(H=2, **kw),
    "c4gqa1": lambda **kw: llama70b_dp8_tp8(H=1, **kw),
    "c5": long_context_tp4_tp8,
    "single": single_promotion,
}


def pool_blocks(w: Workload, slack: float = 1.10, extra: int = 8) -> list:
    """Blocks per GPU pool: an upper bound that needs no layout arithmetic.

    A T-token request never needs more than ceil(T/B) blocks on any GPU at
    any degree (blocks only grow in token capacity), so a GPU that is source
    or destination of a set of requests needs at most the sum of those bounds
    for the sources plus the same for the destinations."""
    need = [0] * w.n_gpus
    for T, s, d in zip(w.T, w.src, w.dst):
        c = -(-T // w.B)
        for g in range(s[0], s[0] + s[1]):
            need[g] += c
        for g in range(d[0], d[0] + d[1]):
            need[g] += c
    return [int(n * slack) + extra for n in need]


def source_tables(w: Workload, counts: list, num_blocks: list, seed: int = 1, window=None,
                  contiguous: bool = False, top: bool = False) -> list:
    """Fragmented source tables: per source group a seeded permutation of the
    IDs [0, window) (default: the whole pool; top: the last `window` IDs of
    the group's smallest pool), consumed in request order, skipping IDs
    already used on any member GPU (groups may overlap).  counts[i] = blocks
    request i holds (computed by the caller's own code)."""
    rng = np.random.default_rng(seed)
    perms, cursor = {}, {}
    used = [np.zeros(n, dtype=bool) for n in num_blocks]
    out = []
    for grp, n in zip(w.src, counts):
        grp = tuple(grp)
        members = range(grp[0], grp[0] + grp[1])
        if grp not in perms:
            nb = min(num_blocks[g] for g in members)
            lo = 0
            if window is not None:
                win = min(nb, int(window[grp] if isinstance(window, dict) else window))
                lo = nb - win if top else 0
                nb = win
            perms[grp] = lo + (np.arange(nb, dtype=np.int32) if contiguous else rng.permutation(nb).astype(np.int32))
            cursor[grp] = 0
        perm, c = perms[grp], cursor[grp]
        ids = []
        while len(ids) < n:
            if c >= len(perm):
                raise ValueError("pool too small for source tables")
            b = int(perm[c])
            c += 1
            if not any(used[g][b] for g in members):
                ids.append(b)
        for g in members:
            used[g][ids] = True
        cursor[grp] = c
        out.append(np.asarray(ids, dtype=np.int32))
    return out


def realistic_pools(w: Workload, n_src: list, n_dst: list, frag: float = 1.25, slack: float = 1.05,
                    seed: int = 1, contiguous: bool = False):
    """Equal-sized pools and fragmented source tables for the benches.

    Each live engine's blocks are scattered (seeded permutation) over the low
    window [0, frag * max per-GPU source blocks) of its pool -- fragmented but
    not spread over the whole pool, as a running engine's are -- and the pool
    adds room for the largest per-GPU destination need.  n_src[i] / n_dst[i]:
    blocks request i holds per rank at its source / destination degree,
    computed by the caller's own code.  Returns (num_blocks, tables)."""
    src_need = [0] * w.n_gpus
    dst_need = [0] * w.n_gpus
    for s, d, a, b in zip(w.src, w.dst, n_src, n_dst):
        for g in range(s[0], s[0] + s[1]):
            src_need[g] += a
        for g in range(d[0], d[0] + d[1]):
            dst_need[g] += b
    if w.extra.get("src_top"):  # per-GPU pools: own source window on top + own destination need below
        win = [int(frag * n) + 16 if n else 0 for n in src_need]
        # forward: window on top, destinations below; reverse: the source need
        # again next to the destination copy
        nb = [max(win[g] + int(slack * dst_need[g]), int(slack * (src_need[g] + dst_need[g]))) + 32
              for g in range(w.n_gpus)]
        windows = {tuple(s): min(win[g] for g in range(s[0], s[0] + s[1])) for s in w.src}
        return nb, source_tables(w, n_src, nb, seed=seed, window=windows, contiguous=contiguous, top=True)
    window = int(frag * max(src_need)) + 16
    nb_all = window + int(slack * max(max(dst_need), max(src_need))) + 32
    nb = [nb_all] * w.n_gpus
    return nb, source_tables(w, n_src, nb, seed=seed, window=window, contiguous=contiguous)


# ------------------------------------------------------------ content hashing
_M32 = 0xFFFFFFFF
_K1, _K2, _K3, _K4 = 0x5BD1E995, 0x27D4EB2F, 0x165667B1, 0x2C1B3C6D


def hash32_np(gpu: int, word: np.ndarray, seed: int = 2) -> np.ndarray:
    """uint32 hash of (seed, gpu, word index).  Products stay < 2^63."""
    w = np.asarray(word, dtype=np.int64)
    lo = w & _M32
    hi = w >> 32
    x = (lo * _K1) & _M32
    x ^= (hi * _K2 + gpu * _K3 + seed * 977) & _M32
    x ^= x >> 15
    x = (x * _K4) & _M32
    x ^= x >> 13
    x = (x * _K1) & _M32
    x ^= x >> 16
    return x.astype(np.uint32)


def fill_hash_np(pool_u8: np.ndarray, gpu: int, seed: int = 2) -> None:
    """Fill a host pool (uint8, size % 4 == 0) with the content hash."""
    w = pool_u8.view(np.uint32)
    step = 1 << 24
    for s in range(0, w.size, step):
        e = min(w.size, s + step)
        w[s:e] = hash32_np(gpu, np.arange(s, e, dtype=np.int64), seed)


def hash32_torch(gpu, word, seed: int = 2):
    """Device twin of hash32_np: int32 tensor of the uint32 hash bits.
    gpu: int or int64 tensor broadcastable to word (int64 tensor)."""
    import torch
    lo = word & _M32
    hi = word >> 32
    x = (lo * _K1) & _M32
    x ^= (hi * _K2 + gpu * _K3 + seed * 977) & _M32
    x ^= x >> 15
    x = (x * _K4) & _M32
    x ^= x >> 13
    x = (x * _K1) & _M32
    x ^= x >> 16
    x = torch.where(x >= (1 << 31), x - (1 << 32), x)
    return x.to(torch.int32)


def fill_hash_torch(pool, gpu: int, seed: int = 2, chunk: int = 1 << 26) -> None:
    """Fill a device (or CPU) torch uint8 pool with the same hash, in place.
    torch int64 arithmetic wraps identically; all products stay < 2^63."""
    import torch
    w = pool.reshape(-1).view(torch.int32)
    n = w.numel()
    dev = pool.device
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = torch.arange(s, e, dtype=torch.int64, device=dev)
        w[s:e] = hash32_torch(gpu, idx, seed)
        del idx
