"""Fixed per-launch cost of kv_paged_decode: graph replays of 640 launches on
a tiny problem (n requests x T tokens, 1 KV head, 8 query heads) -- what a
launch costs when it moves (almost) nothing -- serialized and with
KV_DECODE_AFTER_DECODE (consecutive launches overlapped)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_22593_b200 import flykv as F  # noqa: E402

g = F.geometry(1, 1, 128, 16, 2)
dev = "cuda:0"
for after, n, T in [(a_, n_, t_) for a_ in (False, True) for n_, t_ in ((1, 16), (1, 512), (64, 16), (64, 512), (64, 2048))]:
    nblk = (T + 15) // 16
    layer = torch.zeros(n * nblk * 2 * 16 * 128 + 16, dtype=torch.bfloat16, device=dev)
    rp = torch.arange(0, n * nblk + 1, nblk, dtype=torch.int32, device=dev)
    ids = torch.arange(n * nblk, dtype=torch.int32, device=dev)
    meta = torch.tensor([[i, 16, 1, 0] for i in range(n)], dtype=torch.int32, device=dev)
    lens = torch.full((n,), T, dtype=torch.int32, device=dev)
    q = torch.randn((n, 8, 128), device=dev).to(torch.bfloat16)
    out = torch.empty((n, 8, 128), dtype=torch.float32, device=dev)
    s = torch.cuda.Stream()
    F.kv_paged_decode(g, layer.data_ptr(), n, rp, ids, meta, lens, 8, q, out, 0.1, T, s)
    s.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        for _ in range(640):
            F.kv_paged_decode(g, layer.data_ptr(), n, rp, ids, meta, lens, 8, q, out, 0.1, T, s, after_decode=after)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 5 / 640 * 1e3
    mb = n * T * 512 / 1e6
    mode = "after_decode" if after else "serialized  "
    print(f"{mode} n={n:3d} T={T:5d}: {us:7.2f} us per launch, {mb:7.2f} MB K/V -> {mb / us * 1e3:7.1f} GB/s")
