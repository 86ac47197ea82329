"""ctypes wrapper around the C oracle (oracle/kv_oracle.c).

ORACLE -- TEST INFRASTRUCTURE ONLY.  Only tests/, ``__graft_entry__.smoke()``
and bench.py's ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  It never imports anything from ``paper_2602_22593_b200`` and the
product never imports it.

Every function forwards to the plain C definition in kv_oracle.c, whose
header cites the paper passages (Eq.2, Eq.3, M_block eq.
P:338-340, Eq.1) and the DESIGN.md readings it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kv_oracle.c")
_LIB = os.path.join(_HERE, "liboracle_kv.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with plain gcc (no CUDA, no shared headers)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class _Geom(C.Structure):
    _fields_ = [("L", C.c_int32), ("H", C.c_int32), ("d", C.c_int32),
                ("B", C.c_int32), ("e", C.c_int32)]


@dataclass(frozen=True)
class Geom:
    L: int
    H: int
    d: int
    B: int
    e: int = 2

    def c(self) -> _Geom:
        return _Geom(self.L, self.H, self.d, self.B, self.e)


_P32 = C.POINTER(C.c_int32)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        G = C.POINTER(_Geom)
        for name in ("or_h_loc", "or_block_tokens", "or_replicas"):
            getattr(L, name).argtypes = [G, C.c_int32]
            getattr(L, name).restype = C.c_int32
        L.or_block_bytes.argtypes = [G]
        L.or_block_bytes.restype = C.c_int64
        L.or_num_blocks.argtypes = [G, C.c_int32, C.c_int32]
        L.or_num_blocks.restype = C.c_int32
        L.or_owner_rank.argtypes = [G, C.c_int32, C.c_int32, C.c_int32]
        L.or_owner_rank.restype = C.c_int32
        L.or_local_head.argtypes = [G, C.c_int32, C.c_int32]
        L.or_local_head.restype = C.c_int32
        L.or_first_head.argtypes = [G, C.c_int32, C.c_int32]
        L.or_first_head.restype = C.c_int32
        L.or_locate.argtypes = [G, C.c_int32, C.c_int32, _P32, C.c_int32, C.c_int32,
                                C.c_int32, C.c_int32, _P32, C.POINTER(C.c_int64)]
        L.or_locate.restype = None
        L.or_locate_rid.argtypes = [G, C.c_int32, C.c_int32, _P32, _P32, C.c_int32, C.c_int32,
                                    C.c_int32, C.c_int32, _P32, C.POINTER(C.c_int64)]
        L.or_locate_rid.restype = None
        L.or_switch.argtypes = [G, C.c_int32, _P32, C.POINTER(C.c_void_p), C.c_int32, C.POINTER(C.c_void_p),
                                C.c_int32, _P32, _P32, _P32, _P32, _P32, _P32, _P32,
                                C.POINTER(C.c_void_p), C.POINTER(C.c_void_p), _P32, _P32, C.c_int32]
        L.or_switch.restype = C.c_int32
        L.or_tables.argtypes = [G, C.c_int32, C.c_int32, _P32, _P32, C.POINTER(C.c_void_p), _P32, _P32, _P32, _P32,
                                _P32]
        L.or_tables.restype = C.c_int32
        _P64 = C.POINTER(C.c_int64)
        L.or_atom_map.argtypes = [G, _P32, C.c_int32, C.c_int32, C.c_int32, _P32, _P32, C.c_int32, C.c_int32,
                                  _P32, _P32, _P32, _P64, _P32, _P64]
        L.or_atom_map.restype = C.c_int64
    return _lib


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(_P32)


# ---------------------------------------------------------------- layout math
def h_loc(g: Geom, p: int) -> int:
    return lib().or_h_loc(C.byref(g.c()), p)


def block_tokens(g: Geom, p: int) -> int:
    return lib().or_block_tokens(C.byref(g.c()), p)


def block_bytes(g: Geom) -> int:
    return lib().or_block_bytes(C.byref(g.c()))


def num_blocks(g: Geom, T: int, p: int) -> int:
    return lib().or_num_blocks(C.byref(g.c()), T, p)


def replicas(g: Geom, p: int) -> int:
    return lib().or_replicas(C.byref(g.c()), p)


def owner_rank(g: Geom, p: int, h: int, j: int = 0) -> int:
    return lib().or_owner_rank(C.byref(g.c()), p, h, j)


def first_head(g: Geom, p: int, r: int) -> int:
    return lib().or_first_head(C.byref(g.c()), p, r)


def locate(g: Geom, g0: int, p: int, tab, kv: int, h: int, t: int, j: int = 0, rid=None):
    """(gpu, byte offset inside that GPU's layer region) of token t of head h;
    rid = rank IDs of the group's members (None = identity)."""
    tab = _i32(tab)
    gpu = C.c_int32()
    off = C.c_int64()
    r = _i32(rid) if rid is not None else None
    lib().or_locate_rid(C.byref(g.c()), g0, p, _ptr(r) if r is not None else None, _ptr(tab), kv, h, t, j,
                        C.byref(gpu), C.byref(off))
    return gpu.value, off.value


def _rid_array(rids):
    """ctypes array of int32* (NULL = identity) + keep-alive list."""
    keep = [(_i32(r) if r is not None else None) for r in rids]
    arr = (C.c_void_p * max(len(keep), 1))(*[(k.ctypes.data if k is not None else None) for k in keep])
    return arr, keep


# ---------------------------------------------------------------- the switch
@dataclass
class Req:
    T: int
    src: tuple  # (first_gpu, degree)
    src_ids: list
    dst: tuple  # (first_gpu, degree)
    src_rid: list = None  # rank IDs of the source group's members (None = identity)
    dst_rid: list = None


def switch(g: Geom, pools: list, held: list, reqs: list, copy: bool = True):
    """Run the oracle switch in place.

    pools[gpu]: contiguous uint8 array of L*num_blocks*M bytes ([L][nb][M]),
                or None when copy=False (allocation/release only).
    held[gpu]:  uint8 array [num_blocks], 1 = held by a live request.
    Returns (status, dst_tables as list of np.int32 arrays).
    """
    M = block_bytes(g)
    if copy:
        nb = _i32([p.size // (g.L * M) for p in pools])
        for p, n in zip(pools, nb):
            assert p.dtype == np.uint8 and p.flags.c_contiguous and p.size == g.L * int(n) * M
    else:
        nb = _i32([h.size for h in held])
    for hb, n in zip(held, nb):
        assert hb.dtype == np.uint8 and hb.flags.c_contiguous and hb.size == int(n)
    n = len(reqs)
    T = _i32([r.T for r in reqs])
    sg0 = _i32([r.src[0] for r in reqs])
    sp = _i32([r.src[1] for r in reqs])
    dg0 = _i32([r.dst[0] for r in reqs])
    dp = _i32([r.dst[1] for r in reqs])
    sptr = _i32(np.concatenate([[0], np.cumsum([len(r.src_ids) for r in reqs])]) if n else [0])
    sids = _i32(np.concatenate([np.asarray(r.src_ids, dtype=np.int64) for r in reqs]) if n else [])
    if sids.size == 0:
        sids = _i32([0])
    cap = int(sum(int(n_) for n_ in nb) * 1 + sptr[-1] + 16)
    cap = max(cap, 1)
    dptr = np.zeros(n + 1, dtype=np.int32)
    dids = np.zeros(cap, dtype=np.int32)
    pool_ptrs = (C.c_void_p * len(held))(*([p.ctypes.data for p in pools] if copy else [0] * len(held)))
    held_ptrs = (C.c_void_p * len(held))(*[h.ctypes.data for h in held])
    srid, k1 = _rid_array([r.src_rid for r in reqs])
    drid, k2 = _rid_array([r.dst_rid for r in reqs])
    st = lib().or_switch(C.byref(g.c()), len(held), _ptr(nb), pool_ptrs, int(copy), held_ptrs, n,
                         _ptr(T), _ptr(sg0), _ptr(sp), _ptr(sptr), _ptr(sids), _ptr(dg0), _ptr(dp),
                         srid, drid, _ptr(dptr), _ptr(dids), cap)
    tabs = [dids[dptr[i]:dptr[i + 1]].copy() for i in range(n)] if st == 0 else None
    return st, tabs


def tables(g: Geom, gpu: int, reqs: list, dst_tabs: list):
    """Per-GPU CSR block table after the switch: (req_ptr, ids, meta[n,4])."""
    n = len(reqs)
    dg0 = _i32([r.dst[0] for r in reqs] or [0])
    dp = _i32([r.dst[1] for r in reqs] or [1])
    dptr = _i32(np.concatenate([[0], np.cumsum([len(t) for t in dst_tabs])]) if n else [0])
    dids = _i32(np.concatenate([np.asarray(t, dtype=np.int64) for t in dst_tabs]) if n and dptr[-1] else [0])
    req_ptr = np.zeros(n + 1, dtype=np.int32)
    ids = np.zeros(max(int(dptr[-1]), 1), dtype=np.int32)
    meta = np.zeros(4 * max(n, 1), dtype=np.int32)
    drid, keep = _rid_array([r.dst_rid for r in reqs])
    nres = lib().or_tables(C.byref(g.c()), gpu, n, _ptr(dg0), _ptr(dp), drid, _ptr(dptr), _ptr(dids),
                           _ptr(req_ptr), _ptr(ids), _ptr(meta))
    return req_ptr[:nres + 1].copy(), ids[:req_ptr[nres]].copy(), meta[:4 * nres].reshape(nres, 4).copy()


def atom_map(g: Geom, num_blocks, T: int, src, tab0, dst, tab1, src_rid=None, dst_rid=None):
    """All atom copies of one request: arrays (src_gpu, src_off, dst_gpu, dst_off)."""
    nb = _i32(num_blocks)
    C_ = -(-T // g.B)
    n = g.L * 2 * g.H * C_ * replicas(g, dst[1])
    sg = np.zeros(max(n, 1), dtype=np.int32)
    dg = np.zeros(max(n, 1), dtype=np.int32)
    so = np.zeros(max(n, 1), dtype=np.int64)
    do = np.zeros(max(n, 1), dtype=np.int64)
    t0, t1 = _i32(tab0 if len(tab0) else [0]), _i32(tab1 if len(tab1) else [0])
    P64 = C.POINTER(C.c_int64)
    r0 = _i32(src_rid) if src_rid is not None else None
    r1 = _i32(dst_rid) if dst_rid is not None else None
    m = lib().or_atom_map(C.byref(g.c()), _ptr(nb), T, src[0], src[1], _ptr(r0) if r0 is not None else None, _ptr(t0),
                          dst[0], dst[1], _ptr(r1) if r1 is not None else None, _ptr(t1),
                          _ptr(sg), so.ctypes.data_as(P64), _ptr(dg), do.ctypes.data_as(P64))
    assert m == n
    return sg[:n], so[:n], dg[:n], do[:n]
