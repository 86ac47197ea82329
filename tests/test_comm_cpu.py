"""Communicator pool and replicated planning, world_size 2 and 4 over gloo on
CPU (no GPU): aligned-group enumeration, eager construction and
O(1) lookup, and every rank building the identical plan from the
globally agreed request order, including the kernels' mixed work
order -- the property the one-process-per-GPU path relies on."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_22593_b200 import comm


def test_enumerate_groups_paper_example():
    assert comm.enumerate_tp_groups(4, [2, 4]) == [(0, 1), (2, 3), (0, 1, 2, 3)]
    assert len(comm.enumerate_tp_groups(8, [2, 4, 8])) == 7
    assert comm.enumerate_tp_groups(2, []) == []
    with pytest.raises(ValueError):
        comm.enumerate_tp_groups(4, [3])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_22593_b200 import flykv as F
        import synth
        pool = comm.CommunicatorPool(world, [2, 4], backend="gloo")
        out = {"keys": sorted(pool.groups.keys()), "init_s": pool.init_seconds,
               "host_bytes_per_group": pool.host_bytes_per_group}
        import time as _t
        t0 = _t.perf_counter()
        for _ in range(10000):
            pool.get((0, 1))
        out["lookup_us"] = (_t.perf_counter() - t0) / 10000 * 1e6
        try:
            pool.get((1, 2))
            out["unaligned"] = "found"
        except comm.UnknownGroup:
            out["unaligned"] = "UnknownGroup"
        out["cover"] = pool.covering([(0, 1), (1, 1)])
        out["cover2"] = pool.covering([(2, 1), (0, 2)])
        # replicated allocator + identical plan on every rank (fake pointers)
        w = synth.dp_to_tp(world, 12, L=2, H=8, d=64, B=16, lo=10, hi=300)
        g = F.geometry(w.L, w.H, w.d, w.B, w.e)
        n0 = [F.kv_blocks_for(g, T, s[1]) for T, s in zip(w.T, w.src)]
        n1 = [F.kv_blocks_for(g, T, d[1]) for T, d in zip(w.T, w.dst)]
        nb, tabs = synth.realistic_pools(w, n0, n1)
        bases = [[(1 << 40) + (r << 36) + (l << 30) for l in range(w.L)] for r in range(world)]
        cache = F.KVCache(g, nb, bases, (2, 4))
        for s_, ids in zip(w.src, tabs):
            cache.reserve(s_, ids)
        plan = F.kv_plan_switch(cache, [(i, T, s_, ids, d) for i, (T, s_, d, ids) in
                                        enumerate(zip(w.T, w.src, w.dst, tabs))])
        digest = np.concatenate(plan.dst_tables()).astype(np.int64)
        st, mat = plan.stats()
        # the kernels' work order too: every rank can model (or check) every sender's schedule
        wo = np.concatenate([plan.work_order(x).reshape(-1) for x in range(world)]).astype(np.int64)
        mine = (int(digest.sum()), int((digest * np.arange(digest.size)).sum()), int(mat.sum()),
                int((wo * (np.arange(wo.size) % 9973 + 1)).sum()), int(st["n_buckets"]), int(st["n_atom_slots"]))
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        out["identical_plans"] = all(v == allv[0] for v in allv)
        # a barrier on a pooled subgroup
        sub = pool.get((0, 1)) if rank < 2 else pool.get((2, 3))
        dist.barrier(group=sub)
        out["ok"] = True
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_pool_and_replicated_plans_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        o = res[r]
        assert o["ok"] and o["identical_plans"]
        assert o["unaligned"] == "UnknownGroup"
        assert o["cover"] == (0, 1)
        assert o["lookup_us"] < 50          # O(1) dict lookup
        assert o["host_bytes_per_group"] is not None and o["host_bytes_per_group"] < 64e6
        if world == 4:
            assert o["keys"] == [(0, 1), (0, 1, 2, 3), (2, 3)]
            assert o["cover2"] == (0, 1, 2, 3)


def _fd_worker(rank, world, port, tmpdir, q):
    import tempfile
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # each rank opens its own file and sends its descriptor to every other rank
        path = os.path.join(tmpdir, f"f{rank}")
        with open(path, "w") as f:
            f.write(f"rank {rank}")
        fd = os.open(path, os.O_RDONLY)
        got = comm.share_fds({r: fd for r in range(world) if r != rank}, rank,
                             {r: True for r in range(world) if r != rank}, "test")
        os.close(fd)
        seen = {}
        for src, rfd in got.items():   # pread: the receivers share one open file description
            seen[src] = os.pread(rfd, 64, 0).decode()
            os.close(rfd)
        q.put((rank, seen))
    finally:
        dist.destroy_process_group()


def test_share_fds_gloo():
    """The NVLS path's descriptor passing (comm.share_fds: SCM_RIGHTS over
    abstract AF_UNIX sockets, the transport of kv_pool_export / kv_mc_create
    handles) on 3 gloo ranks: every rank receives a working descriptor of
    every other rank's file."""
    import tempfile
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    with tempfile.TemporaryDirectory() as td:
        procs = [ctx.Process(target=_fd_worker, args=(r, world, port, td, q)) for r in range(world)]
        for p in procs:
            p.start()
        res = dict(q.get(timeout=120) for _ in range(world))
        for p in procs:
            p.join(timeout=60)
    for r in range(world):
        assert res[r] == {s: f"rank {s}" for s in range(world) if s != r}


def _hb_worker(rank, world, port, q):
    import time as _t
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        keys = [(0, 1), (2, 3), (0, 1, 2, 3)]
        hb = comm.HostBarrier(rank, world, keys)
        out = {"outside": hb.arm((2, 3) if rank < 2 else (0, 1)) is None}
        # a member that arrives late holds the others: ranks 1 and 3 sleep 0.3 s
        # before their subgroup barrier, so 0 and 2 leave it no earlier
        fn = hb.arm((0, 1) if rank < 2 else (2, 3))
        t0 = _t.perf_counter()
        if rank % 2:
            _t.sleep(0.3)
        fn()
        out["held_s"] = _t.perf_counter() - t0
        hb.arm((0, 1, 2, 3))()
        out["ok"] = True
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_host_barrier_gloo():
    """comm.HostBarrier (a5 for ranks sharing one GPU) on 4 gloo ranks: the
    callable arm(key) hands to kv_switch_range_host is a barrier over the
    key's members only (the pooled subgroups), None for a non-member."""
    world = 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_hb_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert res[r]["ok"] and res[r]["outside"]
        assert res[r]["held_s"] >= 0.25


def test_device_barrier_arm_bookkeeping():
    """comm.DeviceBarrier.arm without a device: per key, the k-th barrier's
    target is k x members on the 128-byte line of that key in every
    member's counter buffer; a non-member or a one-member key gets None
    (nothing to wait for)."""
    b = object.__new__(comm.DeviceBarrier)
    b.rank, b.world = 1, 4
    b.keys = [(0, 1), (2, 3), (0, 1, 2, 3)]
    b.slot = {k: i for i, k in enumerate(b.keys)}
    b.count = {k: 0 for k in b.keys}
    b.timeout_ns = 123
    b.status = "status"
    b.bases = [1000 * (r + 1) << 20 for r in range(4)]
    flags, me, target, tmo, st = b.arm((0, 1))
    assert (me, target, tmo, st) == (1, 2, 123, "status")
    assert flags == [b.bases[0], b.bases[1]]
    assert b.arm((0, 1))[2] == 4 and b.arm((0, 1, 2, 3))[2] == 4 and b.arm((0, 1, 2, 3))[2] == 8
    flags4 = b.arm((0, 1, 2, 3))[0]
    assert flags4 == [x + 2 * comm.DeviceBarrier.LINE * 8 for x in b.bases]
    assert b.arm((2, 3)) is None and b.count[(2, 3)] == 0
    b.rank = 0
    b.keys.append((0,))
    b.slot[(0,)] = 3
    b.count[(0,)] = 0
    assert b.arm((0,)) is None


def _share_worker(rank, world, port, same, q):
    import types
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uuid = "GPU-A" if same else f"GPU-{rank}"
        torch.cuda.get_device_properties = lambda dev: types.SimpleNamespace(uuid=uuid, pci_bus_id=0)
        q.put((rank, comm.ranks_share_a_device("cuda:0")))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("same", [True, False])
def test_ranks_share_a_device_gloo(same):
    """comm.make_barrier's test: ranks reporting one GPU UUID share a device
    (-> HostBarrier); distinct UUIDs do not (-> DeviceBarrier)."""
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_share_worker, args=(r, world, port, same, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert all(v is same for v in res.values())
