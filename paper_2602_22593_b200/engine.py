"""KVSwitchEngine: the user-facing switch API over libflykv.so.

One call = one live DP<->TP switch of a set of requests:
  kv_plan_switch (host: validate, allocate, plan; descriptors uploaded once)
  -> kv_reshard  (sm_100a kernel, the hot loop)
  -> kv_remap_block_tables for every pool in one launch (sm_100a kernel;
     commits the plan), into torch tensors the caller can hand to attention
  -> optional read-back of the new block tables to host memory.
flykv.kv_switch / kv_switch_back do the same in one C call with plan-owned
tables; execute_pack_unpack runs the pack -> all-to-all -> unpack variant.
torch supplies device memory and streams only.  Single process: every pool
lives on devices this process can address (virtual ranks on one B200, or
peer-enabled GPUs).  One process per GPU: see comm.py.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

import torch

from . import flykv
from .pools import DevicePools


@dataclass
class GpuTable:
    """Post-switch logical table of one pool."""
    req_ptr: torch.Tensor     # int32 [n_res + 1]
    block_ids: torch.Tensor   # int32 [n_ids]
    meta: torch.Tensor        # int32 [n_res, 4]: plan index, B(p), H_loc, first head


class KVSwitchEngine:
    def __init__(self, geom: flykv.Geometry, num_blocks, device="cuda:0", tp_degrees=(2, 4, 8), fill=None,
                 stream=None):
        self.device = torch.device(device)
        self.pools = DevicePools(geom, num_blocks, self.device, fill=fill)
        self.cache = self.pools.make_cache(tp_degrees)
        # every pool is on this one device: no links to balance, so the
        # kernels visit atoms in plan order (the mixed order, for one
        # process per GPU, measured 0.1-1.4% slower here)
        self.cache.set_work_order(0)
        self.geom = geom
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)

    @property
    def n_gpus(self) -> int:
        return self.cache.n_gpus

    def plan(self, requests) -> flykv.Plan:
        return flykv.kv_plan_switch(self.cache, requests)

    def alloc_tables(self, plan: flykv.Plan, gpus):
        """Separate per-pool table buffers (for per-pool kv_remap_block_tables calls)."""
        out = {}
        for g in gpus:
            n_res, n_ids = plan.resident(g)
            out[g] = GpuTable(torch.empty(n_res + 1, dtype=torch.int32, device=self.device),
                              torch.empty(max(n_ids, 1), dtype=torch.int32, device=self.device),
                              torch.empty((max(n_res, 1), 4), dtype=torch.int32, device=self.device))
        return out

    def alloc_packed(self, plan: flykv.Plan):
        """Packed all-pool outputs of kv_remap_block_tables(gpu=-1) and the
        per-pool views into them: {g: GpuTable}, (req_ptr, block_ids, meta)."""
        off, tot = plan.packed_offsets()        # the library's packed layout (kv_plan_packed_offsets)
        rp = torch.empty(int(tot[0]), dtype=torch.int32, device=self.device)
        ids = torch.empty(max(int(tot[1]), 1), dtype=torch.int32, device=self.device)
        meta = torch.empty(max(int(tot[2]), 4), dtype=torch.int32, device=self.device)
        views = {}
        for g in range(self.n_gpus):
            n_res, n_ids = plan.resident(g)
            r0, i0, m0 = (int(x) for x in off[g])
            views[g] = GpuTable(rp[r0:r0 + n_res + 1], ids[i0:i0 + n_ids], meta[m0:m0 + 4 * n_res].view(-1, 4))
        return views, (rp, ids, meta.view(-1, 4))

    def execute(self, plan: flykv.Plan, gpus=None, tables=None):
        """Reshard every atom (one launch) and remap the tables: by default
        all pools in one launch into packed buffers (returns per-pool views);
        with `tables` (from alloc_tables), one launch per listed pool."""
        with torch.cuda.stream(self.stream):
            flykv.kv_reshard(plan, -1, self.stream)
            if tables is None and gpus is None:
                views, (rp, ids, meta) = self.alloc_packed(plan)
                flykv.kv_remap_block_tables(plan, -1, rp, ids, meta, self.stream)
                self._packed = (rp, ids, meta)
                return views
            tables = tables if tables is not None else self.alloc_tables(plan, gpus)
            for g, t in tables.items():
                flykv.kv_remap_block_tables(plan, g, t.req_ptr, t.block_ids, t.meta, self.stream)
        return tables

    def execute_pack_unpack(self, plan: flykv.Plan, buf=None):
        """The pack -> all-to-all -> unpack alternative (kv_pack / kv_unpack)
        with every pool on this device: one buffer holds chunk (s -> d) at the
        row-major prefix of the plan's byte matrix, so the all-to-all is the
        identity and unpack reads what pack wrote.  Then the all-pool remap.
        buf: optional device uint8 buffer of >= payload bytes."""
        st, mat = plan.stats()
        n = self.n_gpus
        _, _, off = plan.a2a_offsets()      # chunk (s -> d) at off[s, d] of one row-major buffer
        if buf is None:
            buf = torch.empty(max(int(st["payload_bytes"]), 16), dtype=torch.uint8, device=self.device)
        with torch.cuda.stream(self.stream):
            for s_ in range(n):
                if mat[s_].sum():
                    flykv.kv_pack(plan, s_, buf, off[s_], self.stream)
            for d in range(n):
                if mat[:, d].sum():
                    flykv.kv_unpack(plan, d, buf, off[:, d], self.stream)
            views, (rp, ids, meta) = self.alloc_packed(plan)
            flykv.kv_remap_block_tables(plan, -1, rp, ids, meta, self.stream)
            self._packed = (rp, ids, meta)
        return views, buf

    def switch(self, requests, gpus=None, read_back=False):
        """Plan + reshard + remap.  With read_back, the new tables are copied
        to host and the call returns after the switch has completed."""
        plan = self.plan(requests)
        tables = self.execute(plan, gpus)
        host = None
        if read_back:
            host = {}
            with torch.cuda.stream(self.stream):
                if gpus is None:  # packed: three device->host copies for every pool's table
                    rp, ids, meta = (x.to("cpu", non_blocking=True) for x in self._packed)
                    self.stream.synchronize()
                    off, _ = plan.packed_offsets()
                    meta = meta.reshape(-1)
                    for g in range(self.n_gpus):
                        n_res, n_ids = plan.resident(g)
                        r0, i0, m0 = (int(x) for x in off[g])
                        host[g] = (rp[r0:r0 + n_res + 1], ids[i0:i0 + n_ids], meta[m0:m0 + 4 * n_res].view(-1, 4))
                else:
                    for g, t in tables.items():
                        n_res, n_ids = plan.resident(g)
                        host[g] = (t.req_ptr.to("cpu", non_blocking=True),
                                   t.block_ids[:n_ids].to("cpu", non_blocking=True),
                                   t.meta[:n_res].to("cpu", non_blocking=True))
            self.stream.synchronize()
        return plan, tables, host

    def switch_pieces(self, requests, max_wave_bytes: int = 0):
        """Memory-bounded switch that may move a request in block-aligned token
        pieces across waves (kv_plan_pieces, R20): the promotion of one long
        request whose source and destination do not fit side by side.  Each
        wave commits (releasing its pieces' sources) before the next wave is
        planned; the kernels of consecutive waves are stream-ordered.  Returns (final destination table of every
        request = concatenation of its pieces' tables, the wave plans).  The
        schedule and the waves run in one kv_switch_waves call."""
        requests = list(requests)
        parts = [[] for _ in requests]
        # schedule (kv_plan_pieces) and all waves in one C call, one sync
        waves, plans = flykv.kv_switch_waves(self.cache, requests, max_wave_bytes, split=True, stream=self.stream)
        for wave, plan in zip(waves, plans):
            for (i, _, _), tab in zip(wave, plan.dst_tables()):
                parts[i].append(tab)
        tables = [np.concatenate(p).astype(np.int32) if p else np.zeros(0, dtype=np.int32) for p in parts]
        return tables, plans

    def switch_waves(self, requests, max_wave_bytes: int = 0, read_back=False):
        """Memory-bounded switch: waves planned by
        kv_plan_waves; each wave is a full switch whose commit frees its
        sources before the next wave allocates.  Returns [(plan, tables, host)]."""
        requests = list(requests)
        waves = flykv.kv_plan_waves(self.cache, requests, max_wave_bytes)
        out = []
        for a, b in waves:
            out.append(self.switch(requests[a:b], read_back=read_back))
        return out
