"""Paged KV pools in device memory (torch is the allocator: plumbing only).

A pool of GPU g is one uint8 tensor [L, num_blocks, M] (layer-major, R5): the
layer-l region starts at data_ptr() + l*num_blocks*M and holds num_blocks
blocks of M = 2*H*B*d*e bytes (M_block eq. P:338-340).  Several pools may live
on one physical device ("virtual ranks") so multi-rank layouts run on one B200.
"""
from __future__ import annotations

import torch

from . import flykv


class DevicePools:
    def __init__(self, geom: flykv.Geometry, num_blocks, devices, fill=None):
        self.geom = geom
        _, _, self.M = flykv.kv_layout(geom, 1)
        self.num_blocks = [int(n) for n in num_blocks]
        if isinstance(devices, (str, torch.device, int)):
            devices = [devices] * len(self.num_blocks)
        self.devices = [torch.device(d) for d in devices]
        L = geom.num_layers
        self.tensors = []
        for nb, dev in zip(self.num_blocks, self.devices):
            t = torch.empty((L, max(nb, 1), self.M), dtype=torch.uint8, device=dev)
            self.tensors.append(t)
        if fill is not None:
            for g, t in enumerate(self.tensors):
                fill(t, g)

    def layer_base(self):
        L = self.geom.num_layers
        out = []
        for t, nb in zip(self.tensors, self.num_blocks):
            base = t.data_ptr()
            out.append([base + l * max(nb, 1) * self.M for l in range(L)])
        return out

    def nbytes(self) -> int:
        return sum(t.numel() for t in self.tensors)

    def make_cache(self, tp_degrees=(2, 4, 8)) -> flykv.KVCache:
        return flykv.KVCache(self.geom, self.num_blocks, self.layer_base(), tp_degrees)
