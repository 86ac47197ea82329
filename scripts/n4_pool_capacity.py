"""SURVEY 8(f) N4 on one B200 (run through gpurun):

(1) Communicator-pool cost under NCCL ("creating NCCL process groups
    ... can take seconds"; "each PyTorch distributed process group
    consumes ~2 MB of host memory").  One GPU can only form size-1 NCCL
    communicators, so this measures the per-group floor: a world-size-1 NCCL
    process group bound to cuda:0 (eager init), then K groups built eagerly
    with new_group the way CommunicatorPool does, each timed, with host RSS
    and device memory read before and after; plus the first collective on a
    group created lazily (what a switch would pay without the pool) against
    an O(1) lookup in the pool.
(2) A B200 Table-2-style max-context table: the paper's linear
    model max_context(p) = (p*C - W) / kv_bytes_per_token fitted to its two
    static H200 rows, with C rescaled to this GPU's memory (same utilisation
    fraction of total memory) and kv bytes per token from the library's
    kv_layout (Eq.2/Eq.3/M_block).
Writes one JSON object to stdout.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import psutil  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2602_22593_b200 import capacity as cap  # noqa: E402
from paper_2602_22593_b200 import comm  # noqa: E402
from paper_2602_22593_b200 import flykv as F  # noqa: E402



def rss():
    return psutil.Process().memory_info().rss


def pool_cost(k_groups=7):
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29561")
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    torch.cuda.synchronize()
    r0, (f0, _) = rss(), torch.cuda.mem_get_info()
    t0 = time.perf_counter()
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    t_world = time.perf_counter() - t0
    r1, (f1, _) = rss(), torch.cuda.mem_get_info()
    per = []
    groups = []
    for _ in range(k_groups):   # CommunicatorPool's eager new_group, one per pooled key
        a, (fa, _) = rss(), torch.cuda.mem_get_info()
        t = time.perf_counter()
        g = dist.new_group(ranks=[0], backend="nccl")
        x = torch.ones(1, device=dev)
        dist.all_reduce(x, group=g)          # forces the communicator if creation was lazy
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        b, (fb, _) = rss(), torch.cuda.mem_get_info()
        per.append({"seconds": dt, "host_bytes": b - a, "device_bytes": fa - fb})
        groups.append(g)
    pool = {(i,): g for i, g in enumerate(groups)}
    t = time.perf_counter()
    for _ in range(100000):
        pool[(3,)]
    lookup_ns = (time.perf_counter() - t) / 100000 * 1e9
    # the CommunicatorPool class itself (world size 1 has no pooled groups; timing of its constructor)
    t = time.perf_counter()
    comm.CommunicatorPool(1, [2, 4, 8], backend="nccl")
    ctor = time.perf_counter() - t
    hb = sorted(p["host_bytes"] for p in per)
    out = {
        "world": {"seconds": round(t_world, 4), "host_bytes": r1 - r0, "device_bytes": f0 - f1},
        "groups": [{k: (round(v, 5) if isinstance(v, float) else v) for k, v in p.items()} for p in per],
        "group_seconds_median": round(sorted(p["seconds"] for p in per)[len(per) // 2], 5),
        "group_host_bytes_median": hb[len(hb) // 2],
        "group_device_bytes_median": sorted(p["device_bytes"] for p in per)[len(per) // 2],
        "pool_lookup_ns": round(lookup_ns, 1),
        "communicator_pool_ctor_seconds_world1": round(ctor, 6),
        "nccl_version": ".".join(str(x) for x in torch.cuda.nccl.version()),
        "note": "size-1 NCCL communicators (one GPU): the per-group floor; a group over k GPUs adds "
                "k-1 peer connections (NVLink buffers) on top",
    }
    dist.destroy_process_group()
    return out


def capacity_table():
    props = torch.cuda.get_device_properties(0)
    t = cap.table2(props.total_memory)
    t.update({"model": "Llama-3-70B (bf16 KV)", "device": props.name})
    return t


if __name__ == "__main__":
    res = {"capacity": capacity_table()}
    res["nccl_pool"] = pool_cost()
    print(json.dumps(res))
