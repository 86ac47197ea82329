"""One process per GPU, peer pools mapped through CUDA IPC, each process's
reshard kernel pushing its atoms into the other processes' pools (the N-GPU
launch shape), then the group barrier (a5), then the remap.  A process may
own several consecutive pools (virtual ranks, kv_reshard_range).  Whole pools
are compared with the oracle.

On a 1-GPU box the processes share cuda:0 (CUDA IPC between processes on one
device).  There the barrier is comm.HostBarrier (stream sync + gloo barrier;
kv_switch_range_host for the one-call mode): the device barrier would be
separate launches of different processes spinning on one another on one
device, which nothing co-schedules.  With one GPU per process
(FLYKV_TEST_DEVICE_OF_RANK=1, >= world GPUs) comm.make_barrier picks the
device barrier (kv_group_barrier over IPC-shared counters).  The device
barrier's code itself is checked on one GPU by test_device_barrier_* (its
members emulated as the CTAs of one cooperative launch)."""
import os
import socket
import tempfile

import numpy as np
import pytest

import synth
from oracle import oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

GEO = (3, 8, 128, 16, 2)
GEOS = {"hetero": (2, 8, 128, 16, 2), "dp_tp": (3, 8, 128, 16, 2), "tp_dp": (3, 8, 128, 16, 2), "gqa": (2, 2, 128, 16, 2), "tp_tp": (2, 8, 64, 16, 2),
        "gqa1": (2, 1, 128, 16, 2)}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _geo(kind):
    """rand<seed>: a seeded random geometry (H_kv 1-8) for the fuzz cases."""
    if kind.startswith("rand"):
        rng = np.random.default_rng(90000 + int(kind[4:]))
        return (2, int(rng.choice([1, 2, 4, 8])), int(rng.choice([64, 128])), 16, 2)
    return GEOS[kind]


def _workload(world, kind="dp_tp", v=1):
    """dp_tp: DP_N -> TP_N merge; tp_dp: the split back (round-robin engines);
    gqa: H_kv=2 < N (replication, TP_N > kv_heads); tp_tp: TP2 pairs -> TP_N."""
    L, H, d, B, _ = _geo(kind)
    world = world * v   # pools
    w = synth.dp_to_tp(world, 6 * world, L=L, H=H, d=d, B=B, lo=1, hi=700, seed=4)
    if kind == "tp_dp":
        w = synth.Workload(w.name, L, H, d, B, 2, world, w.T, list(w.dst), list(w.src))
    elif kind.startswith("rand"):   # random merges / splits / lateral moves over every legal degree
        rng = np.random.default_rng(91000 + int(kind[4:]))
        degrees = [p for p in (1, 2, 4, 8) if p <= world and ((p <= H and H % p == 0) or (p > H and p % H == 0))]
        src, dst, T = [], [], []
        for _ in range(int(rng.integers(4, 14))):
            p0, p1 = int(rng.choice(degrees)), int(rng.choice(degrees))
            src.append((int(rng.integers(0, world // p0)) * p0, p0))
            dst.append((int(rng.integers(0, world // p1)) * p1, p1))
            T.append(int(rng.integers(1, 700)))
        w = synth.Workload("rand", L, H, d, B, 2, world, T, src, dst)
    elif kind == "hetero":   # GPU 0 feeds two TP2 groups, the others one TP_world group (mixed-order offsets)
        dst = [(((i // world) % 2) * 2, 2) if i % world == 0 else (0, world) for i in range(len(w.T))]
        w = synth.Workload(w.name, L, H, d, B, 2, world, w.T, list(w.src), dst)
    elif kind == "tp_tp":
        w = synth.Workload(w.name, L, H, d, B, 2, world, w.T, [((i % (world // 2)) * 2, 2) for i in range(len(w.T))],
                           list(w.dst))
    return w


def _rank(rank, world, port, outdir, kind, mode="push", v=1):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_22593_b200 import comm
        from paper_2602_22593_b200 import flykv as F
        w = _workload(world, kind, v)
        g = F.geometry(*_geo(kind))
        _, _, M = F.kv_layout(g, 1)
        n0 = [F.kv_blocks_for(g, T, s[1]) for T, s in zip(w.T, w.src)]
        n1 = [F.kv_blocks_for(g, T, d[1]) for T, d in zip(w.T, w.dst)]
        nb, tabs = synth.realistic_pools(w, n0, n1)
        mine = range(rank * v, (rank + 1) * v)   # the pools this process owns
        dev = int(os.environ.get("FLYKV_TEST_DEVICE_OF_RANK", "0")) and rank or 0
        torch.cuda.set_device(dev)
        vmm = None
        if mode in ("vmm", "nvls"):   # pools in shareable VMM memory, mapped by peers through POSIX handles
            align = 0
            if mode == "nvls":
                ok, align, why = F.mc_supported(w.n_gpus // w.H if w.n_gpus > w.H else 2, w.L * nb[rank] * M)
                assert ok, why
            vmm, bases_v, nbs_v, imported_v = comm.exchange_pools_vmm(w.L * nb[rank] * M, rank, world, w.L, M,
                                                                      nb[rank], dev, align)
            pool = vmm.tensor((1, w.L, nb[rank], M))
        else:
            pool = torch.empty((v, w.L, nb[rank], M), dtype=torch.uint8, device=f"cuda:{dev}")
        for k, gp in enumerate(mine):
            synth.fill_hash_torch(pool[k], gp)
        if w.src[0][1] > w.H and not kind.startswith("rand"):
            raise RuntimeError("replicated sources not used here")   # (random cases: both sides read replica 0, R10)
        torch.cuda.synchronize()
        if mode == "a2a":  # no peer mappings: other pools' addresses are never dereferenced
            bases = [[pool[0, l].data_ptr() if r == rank else (1 << 44) + (r << 36) + (l << 30) for l in range(w.L)]
                     for r in range(world)]
            nbs, imported = nb, []
        elif vmm is not None:
            bases, nbs, imported = bases_v, nbs_v, []
        else:
            bases, nbs, imported = comm.exchange_pools(pool, rank, world, w.L, M)
        cache = F.KVCache(g, nbs, bases, [p for p in (2, 4, 8) if p <= world * v])
        mcs = []
        if mode == "nvls":   # one multicast team per aligned replica group (N2)
            mcs.append(comm.setup_multicast_teams(cache, vmm, rank, world, world // w.H, w.L, M, nb[rank], dev))
        barrier = comm.make_barrier(rank, world, [tuple(range(world))], f"cuda:{dev}", timeout_s=60)
        for s_, ids in zip(w.src, tabs):
            cache.reserve(s_, ids)
        stream = torch.cuda.Stream(f"cuda:{dev}")
        reqs = [(i, T, s_, ids, d) for i, (T, s_, d, ids) in enumerate(zip(w.T, w.src, w.dst, tabs))]
        if mode == "onecall":   # the public one-call API for this process's share (kv_switch_range)
            plan = F.kv_switch_range(cache, reqs, mine.start, mine.stop, barrier.arm(tuple(range(world))), stream)
        else:
            plan = F.kv_plan_switch(cache, reqs)
        if mode == "onecall":
            pass
        elif mode == "a2a":  # pack -> all_to_all_single (gloo, host copies) -> unpack
            _, mat = plan.stats()
            send_off, recv_off = F.a2a_offsets(plan)
            send = torch.empty(max(int(mat[rank].sum()), 16), dtype=torch.uint8, device="cuda:0")
            F.kv_pack(plan, rank, send, send_off[rank], stream)
            stream.synchronize()
            recv_h = torch.empty(int(mat[:, rank].sum()), dtype=torch.uint8)
            dist.all_to_all_single(recv_h, send[:int(mat[rank].sum())].cpu(), [int(x) for x in mat[:, rank]],
                                   [int(x) for x in mat[rank]])
            recv = recv_h.to("cuda:0") if recv_h.numel() else torch.empty(16, dtype=torch.uint8, device="cuda:0")
            F.kv_unpack(plan, rank, recv, recv_off[rank], stream)
        else:
            F.kv_reshard_range(plan, mine.start, mine.stop, stream)
        out = {}
        if mode == "onecall":   # tables the call read back (owned pools only)
            for gp in mine:
                rp, ids, meta = plan.host_tables(gp)
                out[gp] = (torch.as_tensor(rp), torch.as_tensor(ids), torch.as_tensor(meta))
        else:   # a5: every process's pushes have landed before anyone remaps
            barrier.wait(tuple(range(world)), stream)
        for gp in (mine if mode != "onecall" else ()):
            n_res, n_ids = plan.resident(gp)
            rp = torch.empty(n_res + 1, dtype=torch.int32, device=f"cuda:{dev}")
            ids = torch.empty(max(n_ids, 1), dtype=torch.int32, device=f"cuda:{dev}")
            meta = torch.empty((max(n_res, 1), 4), dtype=torch.int32, device=f"cuda:{dev}")
            F.kv_remap_block_tables(plan, gp, rp, ids, meta, stream)
            out[gp] = (rp, ids[:n_ids], meta[:n_res])
        # a second barrier on the same counters: nobody reads pools before every
        # process's remap (the test's own hand-off; counts advance to 2 x world)
        barrier.wait(tuple(range(world)), stream)
        stream.synchronize()
        barrier.check()
        for k, gp in enumerate(mine):
            np.save(os.path.join(outdir, f"pool{gp}.npy"), pool[k].cpu().numpy().reshape(-1))
            rp, ids, meta = out[gp]
            np.save(os.path.join(outdir, f"rp{gp}.npy"), rp.cpu().numpy())
            np.save(os.path.join(outdir, f"ids{gp}.npy"), ids.cpu().numpy())
            np.save(os.path.join(outdir, f"meta{gp}.npy"), meta.cpu().numpy())
        dist.barrier()
        barrier.close()
        comm.close_pools(imported)
        for m_ in mcs:
            m_.free()
        if vmm is not None:
            del pool
            for pm in imported_v:
                pm.free()
            dist.barrier()
            vmm.free()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind,mode,v", [(2, "dp_tp", "push", 1), (4, "dp_tp", "push", 1),
                                               (4, "tp_dp", "push", 1), (4, "gqa", "push", 1),
                                               (4, "tp_tp", "push", 1), (2, "dp_tp", "a2a", 1),
                                               (4, "tp_dp", "a2a", 1), (4, "gqa", "a2a", 1),
                                               (4, "tp_tp", "a2a", 1), (8, "dp_tp", "push", 1),
                                               (8, "gqa", "push", 1), (8, "tp_tp", "a2a", 1),
                                               (2, "dp_tp", "push", 4), (4, "dp_tp", "push", 2),
                                               (2, "tp_dp", "push", 2), (2, "gqa", "push", 4),
                                               (2, "dp_tp", "vmm", 1), (4, "gqa", "vmm", 1), (4, "tp_tp", "vmm", 1),
                                               (2, "dp_tp", "onecall", 1), (4, "tp_dp", "onecall", 1),
                                               (2, "gqa", "onecall", 4), (8, "dp_tp", "onecall", 1),
                                               (4, "hetero", "push", 1), (4, "hetero", "onecall", 1),
                                               (2, "hetero", "push", 2)]
                         + [(int(np.random.default_rng(92000 + k).choice([2, 4])), f"rand{k}",
                             ["push", "onecall"][k % 2], int(np.random.default_rng(93000 + k).choice([1, 2])))
                            for k in range(int(os.environ.get("FLYKV_MP_FUZZ_CASES", "4")))])
def test_ipc_push_matches_oracle(world, kind, mode, v):
    """push: every process's reshard kernel (kv_reshard_range over the v
    pools it owns) stores into peer pools (CUDA IPC), then kv_group_barrier.
    a2a: kv_pack into per-destination chunks, all_to_all_single (gloo over
    host copies here; NCCL on GPUs), kv_unpack -- no peer mappings at all.
    vmm: pools as shareable VMM allocations mapped through POSIX handles.
    onecall: the whole share of each process through kv_switch_range (plan,
    push, device barrier, remap, read-back in one C call)."""
    import torch.multiprocessing as mp
    w = _workload(world, kind, v)
    og = O.Geom(*_geo(kind))
    n0 = [O.num_blocks(og, T, s[1]) for T, s in zip(w.T, w.src)]
    n1 = [O.num_blocks(og, T, d[1]) for T, d in zip(w.T, w.dst)]
    nb, tabs = synth.realistic_pools(w, n0, n1)
    with tempfile.TemporaryDirectory() as td:
        ctx = mp.get_context("spawn")
        port = _free_port()
        procs = [ctx.Process(target=_rank, args=(r, world, port, td, kind, mode, v)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(timeout=300)
            assert p.exitcode == 0
        M = O.block_bytes(og)
        pools = []
        for r in range(world * v):
            a = np.zeros(og.L * nb[r] * M, dtype=np.uint8)
            synth.fill_hash_np(a, r)
            pools.append(a)
        held = [np.zeros(n, dtype=np.uint8) for n in nb]
        oreqs = []
        for T, s, d, ids in zip(w.T, w.src, w.dst, tabs):
            for r in range(s[1]):
                held[s[0] + r][ids] = 1
            oreqs.append(O.Req(T, s, list(ids), d))
        st, otabs = O.switch(og, pools, held, oreqs)
        assert st == 0
        for r in range(world * v):
            got = np.load(os.path.join(td, f"pool{r}.npy"))
            assert np.array_equal(got, pools[r]), f"rank {r} pool differs"
            rp, ids, meta = O.tables(og, r, oreqs, otabs)
            assert np.array_equal(np.load(os.path.join(td, f"rp{r}.npy")), rp)
            assert np.array_equal(np.load(os.path.join(td, f"ids{r}.npy")), ids)
            assert np.array_equal(np.load(os.path.join(td, f"meta{r}.npy")), meta)


@pytest.mark.parametrize("n", [1, 2, 4, 8, 64])
def test_device_barrier_emulated_members(n):
    """a5's device barrier (the production arrive/wait code) with n members
    emulated as the CTAs of one cooperative launch: 2000 rounds, each member
    publishes a store before every barrier and checks every member's store
    after it -- no member ever passes early, none times out."""
    F = __import__("paper_2602_22593_b200.flykv", fromlist=["flykv"])
    assert F.group_barrier_selftest(n, 2000) == (0, 0)


def test_device_barrier_absent_member_times_out():
    """A member that never arrives: the others end their wait after the
    timeout (reported, not a hang)."""
    F = __import__("paper_2602_22593_b200.flykv", fromlist=["flykv"])
    err, tmo = F.group_barrier_selftest(4, 3, absent=2, timeout_ns=int(20e6))
    assert (err, tmo) == (0, 3)


def test_device_barrier_prearrived_launch():
    """kv_group_barrier as launched in production (one single-thread kernel
    on the stream), with the other members' arrivals already in the
    counter, so the launch waits on no other kernel: it passes, adds its
    own arrival to every member's counter, and a wrong target times out
    into the status word."""
    F = __import__("paper_2602_22593_b200.flykv", fromlist=["flykv"])
    ctr = torch.zeros(3 * 16, dtype=torch.int64, device="cuda:0")
    ctr[0] = 2   # members 1 and 2 have arrived at barrier 1 on member 0's counter
    status = torch.zeros(1, dtype=torch.int32, device="cuda:0")
    flags = [ctr[16 * m:].data_ptr() for m in range(3)]
    F.kv_group_barrier(flags, 0, 3, int(5e9), status)
    torch.cuda.synchronize()
    assert ctr[0].item() == 3 and ctr[16].item() == 1 and ctr[32].item() == 1 and status.item() == 0
    F.kv_group_barrier(flags, 1, 3, int(20e6), status)   # member 1 only has 2 of 3: times out
    torch.cuda.synchronize()
    assert status.item() == 1 and ctr[16].item() == 2


def test_nvls_multicast_parity():
    """N2 on NVLS hardware: one process per GPU, pools in shareable VMM
    memory bound to one multicast object per replica team, DP -> TP with
    H_kv < world: the kernel writes every replicated
    atom once through the team's multimem mapping.  Whole pools equal the
    oracle.  (H_kv = 1: one team of `world` GPUs.)  Needs >= 2 GPUs whose
    driver creates multicast objects; skips
    with the driver's reason otherwise."""
    F = __import__("paper_2602_22593_b200.flykv", fromlist=["flykv"])
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip(f"NVLS multicast needs >= 2 GPUs ({n} visible)")
    ok, _, why = F.mc_supported(2, 64 << 20)
    if not ok:
        pytest.skip(f"multicast unavailable: {why}")
    world = 4 if n >= 4 else 2
    os.environ["FLYKV_TEST_DEVICE_OF_RANK"] = "1"
    try:
        test_ipc_push_matches_oracle(world, "gqa1", "nvls", 1)
    finally:
        os.environ.pop("FLYKV_TEST_DEVICE_OF_RANK", None)
