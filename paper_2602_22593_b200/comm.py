"""Communicator pool and peer-pool exchange for one process per GPU (a5, a9).

* enumerate_tp_groups / CommunicatorPool: the paper's topology-aware, eagerly
  built pool of process groups: only aligned contiguous segments
  [k*p, (k+1)*p) for p in the supported degrees, created with
  torch.distributed.new_group at startup and kept in a map keyed by the
  member-rank tuple for O(1) retrieval.  torch.distributed is the
  plumbing (NCCL over NVLink on B200; gloo for CPU tests).
* exchange_pools: every rank exports a CUDA IPC handle of its KV pool and maps
  every peer's pool, so the reshard kernel of rank g stores directly into the
  destination pools over NVLink 5 / NVSwitch (fused pack + all-to-all-v +
  unpack: no staging buffers, no NCCL data path).
* DeviceBarrier: the group completion barrier (a5) after the pushes, on the
  device: per-process 64-bit counters in IPC-shared memory, one per pooled
  group, advanced by kv_group_barrier (system-scope release adds + acquire
  spin) -- no host round trip and no collective on the data path.
  HostBarrier: the same interface on the host (stream sync + process-group
  barrier) for ranks that share one GPU, where spinning launches of
  different processes are not co-scheduled; make_barrier picks one.
* A process may own several consecutive pools ("virtual ranks": the 8
  engines of a switch mapped onto fewer GPUs); exchange_pools and the
  barrier work on processes, the plan on pools.
"""
from __future__ import annotations

import os
import socket
import time

import torch
import torch.distributed as dist

from . import flykv


class UnknownGroup(KeyError):
    pass


def _rss():
    try:
        import psutil
        return psutil.Process().memory_info().rss
    except Exception:
        return None


def enumerate_tp_groups(n: int, degrees) -> list:
    """Aligned contiguous segments for every p in degrees:
    N=4, {2,4} -> [(0,1),(2,3),(0,1,2,3)]; the count is sum_p N/p (linear)."""
    out = []
    for p in sorted(set(int(x) for x in degrees)):
        if p < 2 or p > n:
            continue
        if n % p:
            raise ValueError(f"TP degree {p} does not divide {n} engines")
        for k in range(n // p):
            out.append(tuple(range(k * p, (k + 1) * p)))
    return out


class CommunicatorPool:
    """Eager map  member-rank tuple -> process group."""

    def __init__(self, world_size: int, degrees=(2, 4, 8), backend=None, eager=True):
        self.world_size = world_size
        self.keys = enumerate_tp_groups(world_size, degrees)
        self.groups = {}
        self.init_seconds = 0.0
        self.host_bytes_per_group = None   # measured RSS growth per group (P:434 quotes ~2 MB)
        if eager:
            rss0 = _rss()
            t0 = time.perf_counter()
            for k in self.keys:  # every rank calls new_group for every group (collective)
                self.groups[k] = dist.new_group(ranks=list(k), backend=backend)
            self.groups[tuple(range(world_size))] = self.groups.get(tuple(range(world_size)), dist.group.WORLD)
            self.init_seconds = time.perf_counter() - t0
            if self.keys and rss0 is not None:
                self.host_bytes_per_group = max(0, _rss() - rss0) / len(self.keys)

    def get(self, ranks):
        """O(1) lookup; unaligned or unknown tuples are scheduler bugs."""
        key = tuple(ranks)
        try:
            return self.groups[key]
        except KeyError:
            raise UnknownGroup(key) from None

    def covering(self, groups) -> tuple:
        """Smallest pooled group covering every (first_gpu, degree) given (R12)."""
        lo = min(g[0] for g in groups)
        hi = max(g[0] + g[1] for g in groups)
        p = 1
        while p < self.world_size and not (lo // p == (hi - 1) // p):
            p *= 2
        first = (lo // p) * p
        key = tuple(range(first, first + p))
        if p == 1:
            return key
        return key if key in self.groups else tuple(range(self.world_size))


def exchange_pools(local: torch.Tensor, rank: int, world: int, L: int, M: int, group=None):
    """All-gather IPC handles of every process's pools and map the peers'.
    local: [L, nb, M] (one pool per process) or [v, L, nb, M] (v consecutive
    pools per process: process r owns pools [r*v, (r+1)*v)).  Returns
    (layer_base [world*v][L] pointers usable on this device, num_blocks
    [world*v], imported [(ptr, offset)] to close later)."""
    v = 1 if local.dim() == 3 else int(local.shape[0])
    nb = int(local.shape[-2])
    handle, off = flykv.ipc_export(local.data_ptr())
    mine = (handle, off, nb, v, local.data_ptr(), os.getpid())
    allv = [None] * world
    dist.all_gather_object(allv, mine, group=group)
    bases, nbs, imported = [], [], []
    for r, (h, o, n, vr, p, pid) in enumerate(allv):
        if r == rank:
            base = local.data_ptr()
        else:
            base = flykv.ipc_import(h, o)
            imported.append((base, o))
        for k in range(vr):
            pb = base + k * L * n * M
            bases.append([pb + l * n * M for l in range(L)])
            nbs.append(n)
    return bases, nbs, imported


# ------------------------------------------------ file-descriptor passing
def _sock_name(tag: str, rank: int) -> str:
    """Abstract-namespace AF_UNIX address (no filesystem entry)."""
    return f"\0flykv-{os.environ.get('MASTER_PORT', '0')}-{tag}-{rank}"


def share_fds(fds_to_send: dict, rank: int, sources: dict, tag: str, group=None, timeout_s: float = 120.0):
    """Send each fd in fds_to_send {dest_rank: fd} to that rank and receive
    one fd from every rank in sources {src_rank: True} over AF_UNIX SCM_RIGHTS
    (the POSIX handles of kv_pool_export / kv_mc_create).  Collective over
    the process group (two barriers).  Returns {src_rank: received fd}."""
    import socket
    import threading
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind(_sock_name(tag, rank))
    srv.listen(max(len(sources), 1))
    srv.settimeout(timeout_s)        # a peer that never connects fails loudly, never hangs
    got = {}

    def serve():
        for _ in range(len(sources)):
            try:
                conn, _ = srv.accept()
            except OSError:
                return
            with conn:
                conn.settimeout(timeout_s)
                msg, fds, _, _ = socket.recv_fds(conn, 16, 1)
                got[int(msg.decode())] = fds[0]
    th = threading.Thread(target=serve)
    th.start()
    dist.barrier(group=group)          # every server is listening
    for dst, fd in fds_to_send.items():
        c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        c.settimeout(timeout_s)
        c.connect(_sock_name(tag, dst))
        socket.send_fds(c, [str(rank).encode()], [fd])
        c.close()
    th.join()
    srv.close()
    if set(got) != set(sources):
        raise RuntimeError(f"share_fds({tag}): rank {rank} received from {sorted(got)}, expected {sorted(sources)}")
    dist.barrier(group=group)
    return got


def exchange_pools_vmm(nbytes: int, rank: int, world: int, L: int, M: int, nb: int, device: int, align: int = 0,
                       group=None):
    """The NVLS-capable counterpart of exchange_pools: every process's pool is
    one shareable physical allocation (kv_pool_alloc), and peers map it
    through its POSIX handle (kv_pool_export -> SCM_RIGHTS -> kv_pool_import)
    instead of CUDA IPC.  One pool per process.  Returns (local PoolMem,
    layer_base [world][L], num_blocks [world], [PoolMem imported])."""
    mine = flykv.PoolMem.alloc(device, nbytes, align)
    fds = {r: mine.export_fd() for r in range(world) if r != rank}
    got = share_fds(fds, rank, {r: True for r in range(world) if r != rank}, "pool", group)
    for fd in fds.values():
        flykv.close_fd(fd)
    sizes = [None] * world
    dist.all_gather_object(sizes, mine.nbytes, group=group)
    imported, bases = [], []
    for r in range(world):
        if r == rank:
            base = mine.ptr
        else:
            pm = flykv.PoolMem.import_fd(got[r], sizes[r], device)
            flykv.close_fd(got[r])
            imported.append(pm)
            base = pm.ptr
        bases.append([base + l * nb * M for l in range(L)])
    return mine, bases, [nb] * world, imported


def setup_multicast_teams(cache, pool: "flykv.PoolMem", rank: int, world: int, team_size: int, L: int, M: int,
                          nb: int, device: int, group=None):
    """N2: bind the pools of every aligned replica team of `team_size`
    processes (one pool per process) to one NVLS multicast object and
    register this process's team in the cache (kv_cache_set_multicast).
    Order per the header: leader creates -> fd to members -> import ->
    add_device (all) -> bind (all) -> map.  Returns the Multicast object."""
    lead = rank - rank % team_size
    members = list(range(lead, lead + team_size))
    if rank == lead:
        mc = flykv.Multicast.create(team_size, pool.nbytes)
        send = {r: mc.fd for r in members if r != rank}
        share_fds(send, rank, {}, f"mc{team_size}", group)
    else:
        got = share_fds({}, rank, {lead: True}, f"mc{team_size}", group)
    sizes = [None] * world
    dist.all_gather_object(sizes, mc.nbytes if rank == lead else 0, group=group)
    if rank != lead:
        mc = flykv.Multicast.import_fd(got[lead], sizes[lead], team_size)
        flykv.close_fd(got[lead])
    mc.add_device(device)
    dist.barrier(group=group)          # every member added before any binds
    mc.bind(pool)
    dist.barrier(group=group)
    va = mc.map(device)
    cache.set_multicast((lead, team_size), [va + l * nb * M for l in range(L)], 1)
    if rank == lead and mc.fd >= 0:
        flykv.close_fd(mc.fd)
    return mc


class DeviceBarrier:
    """a5 between processes, on the device (kv_group_barrier).

    Each process owns one 128-byte line per barrier key (a tuple of process
    ranks; keys must be the same list, in the same order, on every process)
    holding a 64-bit counter, exported through CUDA IPC.  wait(key) enqueues
    on the stream: add 1 to every member's counter, then spin until this
    process's counter reaches (barriers on key so far) x members.  Only
    members call wait(key); the count per key advances identically on every
    member because switches are planned identically."""

    LINE = 16  # int64 per key: one 128-byte line each

    def __init__(self, rank: int, world: int, keys, device, timeout_s: float = 60.0, group=None):
        self.rank, self.world = rank, world
        self.keys = [tuple(k) for k in keys]
        self.slot = {k: i for i, k in enumerate(self.keys)}
        self.count = {k: 0 for k in self.keys}
        self.timeout_ns = int(timeout_s * 1e9)
        self.local = torch.zeros(max(len(self.keys), 1) * self.LINE, dtype=torch.int64, device=device)
        self.status = torch.zeros(1, dtype=torch.int32, device=device)
        torch.cuda.synchronize(device)
        handle, off = flykv.ipc_export(self.local.data_ptr())
        allv = [None] * world
        dist.all_gather_object(allv, (handle, off), group=group)
        self.bases, self.imported = [], []
        for r, (h, o) in enumerate(allv):
            if r == rank:
                self.bases.append(self.local.data_ptr())
            else:
                b = flykv.ipc_import(h, o)
                self.imported.append((b, o))
                self.bases.append(b)

    def arm(self, key):
        """Arguments of the next barrier on `key` for a C call that runs it
        itself (kv_switch_range): (flags, self index, target, timeout_ns,
        status), the count advanced; None if this process has no peer in it."""
        key = tuple(key)
        if self.rank not in key or len(key) < 2:
            return None
        self.count[key] += 1
        s = self.slot[key] * self.LINE * 8
        return ([self.bases[m] + s for m in key], key.index(self.rank), self.count[key] * len(key), self.timeout_ns,
                self.status)

    def wait(self, key, stream):
        args = self.arm(key)
        if args is not None:
            flags, me, target, timeout, status = args
            flykv.kv_group_barrier(flags, me, target, timeout, status, stream)

    def check(self):
        """Raise if any wait timed out (a member never arrived)."""
        if int(self.status.item()) != 0:
            raise RuntimeError("kv_group_barrier timed out: a member never arrived")

    def close(self):
        close_pools(self.imported)
        self.imported = []


class HostBarrier:
    """a5 on the host, same interface as DeviceBarrier: wait(key, stream)
    synchronizes the stream (this process's pushes have completed) and then
    runs a process-group barrier over the key's members; arm(key) returns a
    callable for kv_switch_range_host (the library syncs, then calls it).
    For ranks that share one GPU: a device barrier there would be separate
    launches spinning on one another on one device, which nothing
    co-schedules."""

    def __init__(self, rank: int, world: int, keys, group=None):
        self.rank, self.world = rank, world
        self.keys = [tuple(k) for k in keys]
        self.slot = {k: i for i, k in enumerate(self.keys)}
        self.groups = {}
        for k in self.keys:   # new_group is collective: every rank, same order
            self.groups[k] = group if len(k) == world else dist.new_group(list(k))

    def arm(self, key):
        key = tuple(key)
        if self.rank not in key or len(key) < 2:
            return None
        g = self.groups[key]
        return lambda: dist.barrier(group=g)

    def wait(self, key, stream):
        fn = self.arm(key)
        if fn is not None:
            flykv.stream_sync(stream)
            fn()

    def check(self):
        pass

    def close(self):
        pass


def ranks_share_a_device(device, group=None) -> bool:
    """True when two ranks of the job run on the same physical GPU."""
    props = torch.cuda.get_device_properties(device)
    me = (socket.gethostname(), str(getattr(props, "uuid", "")) or f"{props.pci_bus_id}")
    allv = [None] * dist.get_world_size(group)
    dist.all_gather_object(allv, me, group=group)
    return len(set(allv)) < len(allv)


def make_barrier(rank: int, world: int, keys, device, timeout_s: float = 60.0, group=None):
    """a5 for a one-process-per-GPU job: DeviceBarrier when every rank has
    its own GPU; HostBarrier when ranks share one (test mode on a one-GPU
    box)."""
    if ranks_share_a_device(device, group):
        return HostBarrier(rank, world, keys, group)
    return DeviceBarrier(rank, world, keys, device, timeout_s, group)


def close_pools(imported):
    for ptr, off in imported:
        try:
            flykv.ipc_close(ptr, off)
        except Exception:
            pass


def switch_barrier(stream, group=None, nccl=True, device=None, members=None, rank=None):
    """Host-side a5 (comparator / debugging only; the product path is
    DeviceBarrier): NCCL 1-element all_reduce on the switch stream, or stream
    sync + gloo barrier.  Ranks outside `members` (when given) return."""
    if members is not None and rank not in members:
        return
    if nccl:
        with torch.cuda.stream(stream):
            t = torch.ones(1, device=device)
            dist.all_reduce(t, group=group)
    else:
        flykv.stream_sync(stream)
        dist.barrier(group=group)
