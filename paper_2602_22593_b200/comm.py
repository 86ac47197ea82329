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
* switch_barrier: the group completion barrier (a5) after the pushes.
"""
from __future__ import annotations

import os
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
    """All-gather IPC handles of every rank's pool [L, nb, M] and map the
    peers'.  Returns (layer_base [world][L] pointers usable on this device,
    num_blocks [world], imported [(ptr, offset)] to close later)."""
    nb = local.shape[1]
    handle, off = flykv.ipc_export(local.data_ptr())
    mine = (handle, off, int(nb), local.data_ptr(), os.getpid())
    allv = [None] * world
    dist.all_gather_object(allv, mine, group=group)
    bases, nbs, imported = [], [], []
    for r, (h, o, n, p, pid) in enumerate(allv):
        if r == rank:
            base = local.data_ptr()
        else:
            base = flykv.ipc_import(h, o)
            imported.append((base, o))
        bases.append([base + l * n * M for l in range(L)])
        nbs.append(n)
    return bases, nbs, imported


def close_pools(imported):
    for ptr, off in imported:
        try:
            flykv.ipc_close(ptr, off)
        except Exception:
            pass


def switch_barrier(stream, group=None, nccl=True, device=None, members=None, rank=None):
    """a5: every rank's pushes have landed before anyone remaps / reuses.
    NCCL: a 1-element all_reduce enqueued on the switch stream after the
    reshard kernel (device-side; the kernel ends with a system-scope fence).
    gloo (CPU tests, several ranks sharing one device): stream sync + barrier.
    Ranks outside `members` (when given) have nothing to wait for."""
    if members is not None and rank not in members:
        return
    if nccl:
        with torch.cuda.stream(stream):
            t = torch.ones(1, device=device)
            dist.all_reduce(t, group=group)
    else:
        flykv.stream_sync(stream)
        dist.barrier(group=group)
