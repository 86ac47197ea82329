"""Thin ctypes binding of libflykv.so (include/flykv.h).

Argument marshalling only: every step of the re-layout runs in the C++ host
planner and the sm_100a kernels of libflykv.so.  There is no CPU fallback:
importing this module raises if the library is missing.  Pointers may be
passed as ints or as objects exposing ``data_ptr()`` (torch tensors); streams
as ints, ``None`` (legacy default stream) or objects exposing
``cuda_stream`` (torch.cuda.Stream).

Names follow the C ABI: kv_plan_switch, kv_reshard, kv_remap_block_tables,
weight_shard_view (+ the cache/allocator/IPC helpers).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libflykv.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libflykv.so not found at {LIB_PATH}: build it with "
        "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")

_lib = C.CDLL(LIB_PATH)

# ----------------------------------------------------------------- statuses
KV_OK = 0
STATUS_NAMES = {
    0: "KV_OK", 1: "KV_ERR_INVALID_ARG", 2: "KV_ERR_INDIVISIBLE_DEGREE", 3: "KV_ERR_UNKNOWN_GROUP",
    4: "KV_ERR_RANK_OUT_OF_RANGE", 5: "KV_ERR_INDIVISIBLE_EXTENT", 6: "KV_ERR_OUT_OF_BLOCKS",
    7: "KV_ERR_BAD_BLOCK_TABLE", 8: "KV_ERR_DUPLICATE_REQUEST", 9: "KV_ERR_BAD_STATE", 10: "KV_ERR_CUDA",
    11: "KV_ERR_REPLICA_MISMATCH", 12: "KV_ERR_BARRIER",
}


class FlyKVError(RuntimeError):
    """A non-OK kv_status.  `plans`: plans that committed before the error
    (kv_switch*: their sources are released, so they are the caller's only
    record of where those requests now live; host tables via host_tables
    where the read-back completed)."""

    def __init__(self, status: int, msg: str, plans=()):
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))
        self.plans = list(plans)
        super().__init__(f"{self.name}: {msg}")


def _check(status: int):
    if status != KV_OK:
        raise FlyKVError(status, _lib.kv_last_error().decode())


# ----------------------------------------------------------------- structs
class Geometry(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("block_base", C.c_int32), ("elem_bytes", C.c_int32)]


class Group(C.Structure):
    _fields_ = [("first_gpu", C.c_int32), ("degree", C.c_int32)]


class Request(C.Structure):
    _fields_ = [("req_id", C.c_int64), ("num_tokens", C.c_int32), ("src", Group),
                ("src_blocks", C.POINTER(C.c_int32)), ("n_src_blocks", C.c_int32), ("dst", Group),
                ("src_rank_ids", C.POINTER(C.c_int32)), ("dst_rank_ids", C.POINTER(C.c_int32))]


class PlanStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("n_requests", "n_moving", "n_atoms", "n_atom_writes", "atom_bytes",
                                         "payload_bytes", "h2d_bytes", "n_segments", "n_atom_slots",
                                         "n_buckets", "t_plan_ns", "t_enqueue_ns", "t_wait_ns", "t_read_ns")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


KV_W_COLUMN, KV_W_ROW, KV_W_QKV = 0, 1, 2


class WeightDesc(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("rows", C.c_int64), ("cols", C.c_int64), ("ld", C.c_int64),
                ("elem_bytes", C.c_int32), ("kind", C.c_int32), ("num_q_heads", C.c_int32),
                ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32)]


class ViewSegment(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("rows", C.c_int64), ("cols", C.c_int64), ("ld", C.c_int64),
                ("row0", C.c_int64), ("col0", C.c_int64)]


class View(C.Structure):
    _fields_ = [("n_seg", C.c_int32), ("elem_bytes", C.c_int32), ("seg", ViewSegment * 3)]

    def segments(self):
        return [self.seg[k] for k in range(self.n_seg)]


_P = C.c_void_p
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)


def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)


_sig("kv_cache_create", C.c_int, C.POINTER(Geometry), C.c_int32, _I32P, C.POINTER(C.c_void_p), _I32P,
     C.c_int32, C.POINTER(_P))
_sig("kv_cache_destroy", None, _P)
_sig("kv_layout", C.c_int, C.POINTER(Geometry), C.c_int32, _I32P, _I32P, _I64P)
_sig("kv_blocks_for", C.c_int, C.POINTER(Geometry), C.c_int32, C.c_int32, _I32P)
_sig("kv_alloc", C.c_int, _P, Group, C.c_int32, _I32P)
_sig("kv_reserve", C.c_int, _P, Group, _I32P, C.c_int32)
_sig("kv_free", C.c_int, _P, Group, _I32P, C.c_int32)
_sig("kv_free_count", C.c_int, _P, C.c_int32, _I32P)
_sig("kv_held_mask", C.c_int, _P, C.c_int32, C.POINTER(C.c_uint8))
_sig("kv_plan_switch", C.c_int, _P, C.POINTER(Request), C.c_int32, C.POINTER(_P))
_sig("kv_plan_upload", C.c_int, _P, _P)
_sig("kv_reshard", C.c_int, _P, C.c_int32, _P)
_sig("kv_reshard_range", C.c_int, _P, C.c_int32, C.c_int32, _P)
_sig("kv_group_barrier", C.c_int, C.POINTER(C.c_void_p), C.c_int32, C.c_int32, C.c_uint64, C.c_int64, _P, _P)
_sig("kv_plan_resident", C.c_int, _P, C.c_int32, _I32P, _I32P)
_sig("kv_reshard_staged", C.c_int, _P, C.c_int32, _P, C.c_int64, C.c_int32, _P)
_sig("kv_remap_block_tables", C.c_int, _P, C.c_int32, _P, _P, _P, _P)
_sig("kv_switch", C.c_int, _P, C.POINTER(Request), C.c_int32, _P, C.POINTER(_P))
_sig("kv_plan_tables", C.c_int, _P, C.c_int32, C.c_int32, C.POINTER(_I32P), C.POINTER(_I32P), C.POINTER(_I32P))
_sig("kv_switch_back", C.c_int, _P, _P, _P, C.POINTER(_P))
_sig("kv_switch_range", C.c_int, _P, C.POINTER(Request), C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p),
     C.c_int32, C.c_int32, C.c_uint64, C.c_int64, _P, _P, C.POINTER(_P))
HOST_BARRIER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p)
_sig("kv_switch_range_host", C.c_int, _P, C.POINTER(Request), C.c_int32, C.c_int32, C.c_int32, HOST_BARRIER_FN, _P,
     _P, C.POINTER(_P))
_sig("kv_group_barrier_selftest", C.c_int, C.c_int32, C.c_int32, C.c_int32, C.c_int64, _I32P, _I32P)
_sig("kv_switch_multi", C.c_int, _P, C.POINTER(Request), _I32P, C.c_int32, _P, C.POINTER(_P))
_sig("kv_pack", C.c_int, _P, C.c_int32, _P, _I64P, _P)
_sig("kv_unpack", C.c_int, _P, C.c_int32, _P, _I64P, _P)
_sig("kv_plan_dst_tables", C.c_int, _P, _I32P, _I32P)
_sig("kv_plan_commit", C.c_int, _P)
_sig("kv_plan_waves", C.c_int, _P, C.POINTER(Request), C.c_int32, C.c_int64, _I32P, _I32P)
_sig("kv_suggest_rank_ids", C.c_int, _P, C.POINTER(Request), C.c_int32, Group, _I32P)


class Piece(C.Structure):
    _fields_ = [("wave", C.c_int32), ("req", C.c_int32), ("tok0", C.c_int32), ("tok1", C.c_int32)]


_sig("kv_plan_pieces", C.c_int, _P, C.POINTER(Request), C.c_int32, C.c_int64, C.c_int32, C.POINTER(Piece), _I32P)
_sig("kv_switch_waves", C.c_int, _P, C.POINTER(Request), C.c_int32, C.c_int64, C.c_int32, _P, C.c_int32,
     C.POINTER(Piece), _I32P, C.POINTER(_P), _I32P)
_sig("kv_plan_get_stats", C.c_int, _P, C.POINTER(PlanStats), _I64P)
_sig("kv_plan_a2a_offsets", C.c_int, _P, _I64P, _I64P, _I64P)
_sig("kv_plan_packed_offsets", C.c_int, _P, _I32P, _I64P)
_sig("kv_piece_request", C.c_int, C.POINTER(Geometry), C.POINTER(Request), C.c_int32, C.c_int32, C.POINTER(Request))
_sig("kv_plan_destroy", None, _P)
_sig("weight_shard_view", C.c_int, C.POINTER(WeightDesc), C.c_int32, C.c_int32, C.POINTER(View))
_sig("kv_gather_view", C.c_int, C.POINTER(View), _P, _P)
_sig("kv_vmm_granularity", C.c_int, C.c_int32, C.POINTER(C.c_uint64))
_sig("kv_vmm_alloc", C.c_int, C.c_int32, C.c_uint64, C.POINTER(_P), C.POINTER(_P))
_sig("kv_vmm_free", C.c_int, _P)
_sig("weight_view_alias", C.c_int, _P, C.POINTER(View), C.POINTER(_P), C.POINTER(C.c_uint64))
_sig("weight_view_unalias", C.c_int, _P, C.c_uint64)
_sig("kv_paged_decode", C.c_int, C.POINTER(Geometry), _P, C.c_int32, _P, _P, _P, _P, C.c_int32, _P, _P, C.c_float,
     C.c_int32, C.c_int32, _P)
KV_DECODE_AFTER_DECODE = 1
_sig("kv_paged_decode_release", C.c_int, _P)
_sig("kv_ipc_export", C.c_int, _P, C.POINTER(C.c_uint8), C.POINTER(C.c_uint64))
_sig("kv_ipc_import", C.c_int, C.POINTER(C.c_uint8), C.c_uint64, C.POINTER(_P))
_sig("kv_ipc_close", C.c_int, _P, C.c_uint64)
_sig("kv_stream_sync", C.c_int, _P)
_U64P = C.POINTER(C.c_uint64)
_sig("kv_pool_alloc", C.c_int, C.c_int32, C.c_uint64, C.c_uint64, C.POINTER(_P), C.POINTER(_P))
_sig("kv_pool_export", C.c_int, _P, _I32P)
_sig("kv_pool_import", C.c_int, C.c_int32, C.c_uint64, C.c_int32, C.POINTER(_P), C.POINTER(_P))
_sig("kv_pool_free", C.c_int, _P)
_sig("kv_mc_supported", C.c_int, C.c_int32, C.c_uint64, _I32P, _U64P)
_sig("kv_mc_create", C.c_int, C.c_int32, C.c_uint64, C.POINTER(_P), _I32P)
_sig("kv_mc_import", C.c_int, C.c_int32, C.c_uint64, C.c_int32, C.POINTER(_P))
_sig("kv_mc_add_device", C.c_int, _P, C.c_int32)
_sig("kv_mc_bind", C.c_int, _P, _P)
_sig("kv_mc_map", C.c_int, _P, C.c_int32, C.POINTER(_P))
_sig("kv_mc_free", C.c_int, _P)
_sig("kv_close_fd", C.c_int, C.c_int32)
_sig("kv_pool_size", C.c_int, _P, _U64P)
_sig("kv_mc_size", C.c_int, _P, _U64P)
_sig("kv_cache_set_multicast", C.c_int, _P, Group, C.POINTER(_P), C.c_int32)
_sig("kv_strerror", C.c_char_p, C.c_int)
_sig("kv_last_error", C.c_char_p)
_sig("kv_launch_count", C.c_int64)
_sig("kv_set_reshard_impl", C.c_int, C.c_int32, C.c_int32)
_sig("kv_cache_set_work_order", C.c_int, _P, C.c_int32)
_sig("kv_cache_set_strict", C.c_int, _P, C.c_int32)
_sig("kv_verify_replicas", C.c_int, _P, _P, _I64P, C.POINTER(C.c_uint64))
_sig("kv_plan_work_order", C.c_int, _P, C.c_int32, _I32P, _I64P)

EXPORTED = ["kv_cache_create", "kv_cache_destroy", "kv_layout", "kv_blocks_for", "kv_alloc", "kv_reserve",
            "kv_free", "kv_free_count", "kv_held_mask", "kv_plan_switch", "kv_plan_upload", "kv_reshard", "kv_reshard_range", "kv_reshard_staged",
            "kv_pack", "kv_unpack", "kv_switch", "kv_switch_back", "kv_switch_range", "kv_switch_range_host", "kv_switch_multi", "kv_switch_waves", "kv_plan_tables", "kv_plan_resident",
            "kv_remap_block_tables", "kv_plan_dst_tables", "kv_plan_commit", "kv_plan_waves", "kv_plan_pieces",
            "kv_suggest_rank_ids", "kv_plan_get_stats", "kv_plan_a2a_offsets", "kv_piece_request", "kv_plan_packed_offsets",
            "kv_plan_destroy",
            "weight_shard_view", "kv_gather_view", "kv_vmm_granularity", "kv_vmm_alloc", "kv_vmm_free",
            "weight_view_alias", "weight_view_unalias", "kv_paged_decode", "kv_paged_decode_release", "kv_ipc_export", "kv_ipc_import", "kv_ipc_close",
            "kv_group_barrier", "kv_group_barrier_selftest", "kv_stream_sync", "kv_strerror", "kv_last_error", "kv_launch_count", "kv_set_reshard_impl",
            "kv_cache_set_work_order", "kv_plan_work_order", "kv_cache_set_strict", "kv_verify_replicas",
            "kv_pool_alloc", "kv_pool_export", "kv_pool_import", "kv_pool_free", "kv_mc_supported", "kv_mc_create",
            "kv_mc_import", "kv_mc_add_device", "kv_mc_bind", "kv_mc_map", "kv_mc_free", "kv_close_fd",
            "kv_cache_set_multicast", "kv_pool_size", "kv_mc_size"]


# ----------------------------------------------------------------- marshalling
def ptr_of(x) -> int:
    if x is None:
        return 0
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return int(x.data_ptr())
    raise TypeError(f"cannot take a device pointer of {type(x)}")


def stream_of(s) -> int:
    if s is None:
        return 0
    if isinstance(s, int):
        return s
    if hasattr(s, "cuda_stream"):
        return int(s.cuda_stream)
    raise TypeError(f"cannot take a CUDA stream of {type(s)}")


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32).reshape(-1))


def geometry(L: int, H: int, d: int, B: int, e: int = 2) -> Geometry:
    return Geometry(L, H, d, B, e)


def kv_layout(geom: Geometry, degree: int):
    """(H_loc(p), B(p), M) -- Eq.3 / Eq.2 / M_block eq."""
    hl, bt, M = C.c_int32(), C.c_int32(), C.c_int64()
    _check(_lib.kv_layout(C.byref(geom), degree, C.byref(hl), C.byref(bt), C.byref(M)))
    return hl.value, bt.value, M.value


def kv_blocks_for(geom: Geometry, num_tokens: int, degree: int) -> int:
    n = C.c_int32()
    _check(_lib.kv_blocks_for(C.byref(geom), num_tokens, degree, C.byref(n)))
    return n.value


def launch_count() -> int:
    return int(_lib.kv_launch_count())


def set_reshard_impl(impl: int = 0, ctas_per_sm: int = 0):
    """0 default (LDG/STG), 1 LDG/STG, 2 TMA bulk ring (local pools)."""
    _check(_lib.kv_set_reshard_impl(impl, ctas_per_sm))


def strerror(status: int) -> str:
    return _lib.kv_strerror(status).decode()


# ----------------------------------------------------------------- cache
class KVCache:
    """Owns a kv_cache*: per-GPU pools (caller memory) + allocator bitmaps."""

    def __init__(self, geom: Geometry, num_blocks, layer_base, tp_degrees=(2, 4, 8)):
        self.geom = geom
        self.n_gpus = len(num_blocks)
        nb = _i32(num_blocks)
        flat = [ptr_of(p) for row in layer_base for p in row]
        if len(flat) != self.n_gpus * geom.num_layers:
            raise ValueError("layer_base must be [n_gpus][num_layers]")
        self._bases = (C.c_void_p * len(flat))(*flat)
        deg = _i32(tp_degrees) if len(tp_degrees) else _i32([0])
        h = C.c_void_p()
        _check(_lib.kv_cache_create(C.byref(geom), self.n_gpus, nb.ctypes.data_as(_I32P), self._bases,
                                    deg.ctypes.data_as(_I32P), len(tp_degrees), C.byref(h)))
        self._h = h
        self.num_blocks = [int(x) for x in nb]

    def close(self):
        if getattr(self, "_h", None):
            _lib.kv_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def alloc(self, group, n: int) -> np.ndarray:
        out = np.zeros(max(n, 1), dtype=np.int32)
        _check(_lib.kv_alloc(self._h, Group(*group), n, out.ctypes.data_as(_I32P)))
        return out[:n]

    def reserve(self, group, ids):
        ids = _i32(ids)
        _check(_lib.kv_reserve(self._h, Group(*group), ids.ctypes.data_as(_I32P), ids.size))

    def free(self, group, ids):
        ids = _i32(ids)
        _check(_lib.kv_free(self._h, Group(*group), ids.ctypes.data_as(_I32P), ids.size))

    def free_count(self, gpu: int) -> int:
        n = C.c_int32()
        _check(_lib.kv_free_count(self._h, gpu, C.byref(n)))
        return n.value

    def held_mask(self, gpu: int) -> np.ndarray:
        out = np.zeros(max(self.num_blocks[gpu], 1), dtype=np.uint8)
        _check(_lib.kv_held_mask(self._h, gpu, out.ctypes.data_as(C.POINTER(C.c_uint8))))
        return out[:self.num_blocks[gpu]]

    def plan_switch(self, requests) -> "Plan":
        return kv_plan_switch(self, requests)

    def set_strict(self, strict: bool = True):
        """R10 strict mode: kv_switch* verify replicated sources first (kv_cache_set_strict)."""
        _check(_lib.kv_cache_set_strict(self._h, int(bool(strict))))

    def set_multicast(self, team, layer_base, mode: int = 1):
        """Register (or, layer_base None, clear) the NVLS multicast mapping of
        replica team (first_pool, size) -- kv_cache_set_multicast."""
        arr = None
        if layer_base is not None:
            arr = (C.c_void_p * len(layer_base))(*[ptr_of(p) for p in layer_base])
        _check(_lib.kv_cache_set_multicast(self._h, Group(*team), arr, mode))

    def set_work_order(self, order: int):
        """1 = destination-rotated (default), 0 = plan order (kv_cache_set_work_order)."""
        _check(_lib.kv_cache_set_work_order(self._h, order))


# ----------------------------------------------------------------- plan
class Plan:
    def __init__(self, cache: KVCache, handle: C.c_void_p, n_reqs: int):
        self.cache = cache
        self._h = handle
        self.n_reqs = n_reqs

    def destroy(self):
        if getattr(self, "_h", None):
            _lib.kv_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def upload(self, stream=None):
        _check(_lib.kv_plan_upload(self._h, stream_of(stream)))

    def reshard(self, gpu: int = -1, stream=None):
        return kv_reshard(self, gpu, stream)

    def resident(self, gpu: int):
        n, m = C.c_int32(), C.c_int32()
        _check(_lib.kv_plan_resident(self._h, gpu, C.byref(n), C.byref(m)))
        return n.value, m.value

    def remap_block_tables(self, gpu, req_ptr, block_ids, per_req_meta, stream=None):
        return kv_remap_block_tables(self, gpu, req_ptr, block_ids, per_req_meta, stream)

    def commit(self):
        _check(_lib.kv_plan_commit(self._h))

    def dst_tables(self) -> list:
        ptr = np.zeros(self.n_reqs + 1, dtype=np.int32)
        _check(_lib.kv_plan_dst_tables(self._h, ptr.ctypes.data_as(_I32P), None))
        ids = np.zeros(max(int(ptr[-1]), 1), dtype=np.int32)
        _check(_lib.kv_plan_dst_tables(self._h, ptr.ctypes.data_as(_I32P), ids.ctypes.data_as(_I32P)))
        return [ids[ptr[i]:ptr[i + 1]].copy() for i in range(self.n_reqs)]

    def _tables(self, gpu: int, on_device: int):
        rp, ids, meta = _I32P(), _I32P(), _I32P()
        _check(_lib.kv_plan_tables(self._h, gpu, on_device, C.byref(rp), C.byref(ids), C.byref(meta)))
        n_res, n_ids = self.resident(gpu)
        return (C.cast(rp, C.c_void_p).value or 0, C.cast(ids, C.c_void_p).value or 0,
                C.cast(meta, C.c_void_p).value or 0, n_res, n_ids)

    def host_tables(self, gpu: int):
        """(req_ptr, block_ids, meta) of pool gpu after kv_switch, as numpy copies."""
        rp, ids, meta, n_res, n_ids = self._tables(gpu, 0)

        def arr(ptr, n):
            if n == 0:
                return np.zeros(0, dtype=np.int32)
            return np.ctypeslib.as_array(C.cast(ptr, _I32P), shape=(n,)).copy()
        return arr(rp, n_res + 1), arr(ids, n_ids), arr(meta, 4 * n_res).reshape(n_res, 4)

    def device_tables(self, gpu: int):
        """(req_ptr, block_ids, meta, n_resident, n_ids) device pointers (ints) of pool gpu after kv_switch."""
        return self._tables(gpu, 1)

    def stats(self):
        st = PlanStats()
        n = self.cache.n_gpus
        mat = np.zeros(n * n, dtype=np.int64)
        _check(_lib.kv_plan_get_stats(self._h, C.byref(st), mat.ctypes.data_as(_I64P)))
        return st.as_dict(), mat.reshape(n, n)

    def a2a_offsets(self):
        """(send_off, recv_off, packed): int64 [n, n] byte offsets of
        kv_plan_a2a_offsets -- send_off[s] is kv_pack's chunk_off for source
        s, recv_off[d] kv_unpack's for destination d, packed[s, d] the chunk
        (s -> d) in one row-major buffer of every chunk."""
        n = self.cache.n_gpus
        out = [np.zeros(n * n, dtype=np.int64) for _ in range(3)]
        _check(_lib.kv_plan_a2a_offsets(self._h, *(o.ctypes.data_as(_I64P) for o in out)))
        return tuple(o.reshape(n, n) for o in out)

    def packed_offsets(self):
        """(offsets int32 [n, 3], totals int64 [3]) of the packed all-pool
        remap outputs (kv_plan_packed_offsets)."""
        n = self.cache.n_gpus
        off = np.zeros(3 * n, dtype=np.int32)
        tot = np.zeros(3, dtype=np.int64)
        _check(_lib.kv_plan_packed_offsets(self._h, off.ctypes.data_as(_I32P), tot.ctypes.data_as(_I64P)))
        return off.reshape(n, 3), tot

    def work_order(self, gpu: int) -> np.ndarray:
        """[n_pieces, n_gpus + 1] int64: destination bytes per GPU of each of
        `gpu`'s work pieces in kernel order, last column the bytes read."""
        n = self.cache.n_gpus
        k = C.c_int32()
        _check(_lib.kv_plan_work_order(self._h, gpu, C.byref(k), None))
        out = np.zeros((max(k.value, 1), n + 1), dtype=np.int64)
        _check(_lib.kv_plan_work_order(self._h, gpu, C.byref(k), out.ctypes.data_as(_I64P)))
        return out[:k.value]


# numpy twin of the kv_request struct (offsets checked against ctypes below),
# so request lists are marshalled with a few vectorised column writes
_REQ_DTYPE = np.dtype({
    "names": ["req_id", "num_tokens", "src_g0", "src_p", "src_blocks", "n_src_blocks", "dst_g0", "dst_p",
              "src_rank_ids", "dst_rank_ids"],
    "formats": [np.int64, np.int32, np.int32, np.int32, np.uint64, np.int32, np.int32, np.int32, np.uint64,
                np.uint64],
    "offsets": [Request.req_id.offset, Request.num_tokens.offset, Request.src.offset, Request.src.offset + 4,
                Request.src_blocks.offset, Request.n_src_blocks.offset, Request.dst.offset, Request.dst.offset + 4,
                Request.src_rank_ids.offset, Request.dst_rank_ids.offset],
    "itemsize": C.sizeof(Request)})


class _ReqArray:
    """A marshalled request list: .ptr (kv_request*), .n, plus keep-alive."""

    def __init__(self, reqs):
        reqs = list(reqs)
        self.n = len(reqs)
        self.buf = np.zeros(max(self.n, 1), dtype=_REQ_DTYPE)
        self.keep = []
        if self.n == 0:
            self.ptr = C.cast(self.buf.ctypes.data, C.POINTER(Request))
            return
        # all source tables in one contiguous int32 buffer: one pointer fetch,
        # per-request pointers = base + 4 * offset
        tabs = [np.asarray(r[3], dtype=np.int32).reshape(-1) for r in reqs]
        lens = np.fromiter((a.size for a in tabs), dtype=np.int64, count=self.n)
        cat = np.concatenate(tabs) if lens.sum() else np.zeros(1, dtype=np.int32)
        self.keep = [cat]
        base = cat.__array_interface__["data"][0]
        offs = np.zeros(self.n, dtype=np.int64)
        np.cumsum(lens[:-1], out=offs[1:])
        b = self.buf
        b["req_id"] = [r[0] for r in reqs]
        b["num_tokens"] = [r[1] for r in reqs]
        b["src_g0"] = [r[2][0] for r in reqs]
        b["src_p"] = [r[2][1] for r in reqs]
        b["dst_g0"] = [r[4][0] for r in reqs]
        b["dst_p"] = [r[4][1] for r in reqs]
        b["src_blocks"] = np.where(lens > 0, base + 4 * offs, 0).astype(np.uint64)
        b["n_src_blocks"] = lens
        for col, k in (("src_rank_ids", 5), ("dst_rank_ids", 6)):
            ptrs = []
            for r in reqs:
                x = r[k] if len(r) > k else None
                if x is None:
                    ptrs.append(0)
                else:
                    xa = _i32(x)
                    self.keep.append(xa)
                    ptrs.append(xa.ctypes.data)
            b[col] = ptrs
        self.ptr = C.cast(b.ctypes.data, C.POINTER(Request))


def make_requests(reqs) -> _ReqArray:
    """reqs: iterable of (req_id, num_tokens, (g0, p0), src_ids, (g1, p1)
    [, src_rank_ids [, dst_rank_ids]]) -- rank IDs None = identity.
    Returns the marshalled array: .ptr is the kv_request*, .n the count; it
    owns every buffer the pointers refer to."""
    return _ReqArray(reqs)


def kv_plan_switch(cache: KVCache, requests) -> Plan:
    """Validate, allocate and plan a switch (see include/flykv.h)."""
    ra = make_requests(requests)
    h = C.c_void_p()
    _check(_lib.kv_plan_switch(cache._h, ra.ptr, ra.n, C.byref(h)))
    return Plan(cache, h, ra.n)


def kv_switch(cache: KVCache, requests, stream=None) -> Plan:
    """The whole single-process switch in one C call (plan, upload, reshard,
    remap, one table read-back, sync); tables via Plan.host_tables /
    Plan.device_tables."""
    ra = make_requests(requests)
    h = C.c_void_p()
    st = _lib.kv_switch(cache._h, ra.ptr, ra.n, stream_of(stream), C.byref(h))
    plan = Plan(cache, h, ra.n) if h.value else None
    if st != KV_OK:  # a plan returned with an error has committed: hand it over
        raise FlyKVError(st, _lib.kv_last_error().decode(), [plan] if plan is not None else [])
    return plan


def kv_switch_range(cache: KVCache, requests, gpu_lo: int, gpu_hi: int, barrier=None, stream=None) -> Plan:
    """kv_switch for one process of a one-process-per-GPU job owning pools
    [gpu_lo, gpu_hi): plan, upload, push, group barrier, remap of the owned
    pools, one read-back, sync -- one C call.
    barrier: (flags, self_index, target, timeout_ns, status) from
    comm.DeviceBarrier.arm(key) -> kv_switch_range (device barrier); a
    callable from comm.HostBarrier.arm(key) -> kv_switch_range_host (the
    library syncs the stream, then calls it); None when no other process is
    involved."""
    ra = make_requests(requests)
    h = C.c_void_p()
    if callable(barrier):
        err = []

        def _cb(_ctx):
            try:
                barrier()
                return 0
            except Exception as ex:  # reported as KV_ERR_BARRIER; the exception is chained below
                err.append(ex)
                return 1

        st = _lib.kv_switch_range_host(cache._h, ra.ptr, ra.n, gpu_lo, gpu_hi, HOST_BARRIER_FN(_cb), None,
                                       stream_of(stream), C.byref(h))
        plan = Plan(cache, h, ra.n) if h.value else None
        if st != KV_OK:
            raise FlyKVError(st, _lib.kv_last_error().decode(), [plan] if plan is not None else []) from (
                err[0] if err else None)
        return plan
    if barrier is None:
        arr, n_m, me, tgt, tmo, status = None, 0, 0, 0, 1, None
    else:
        flags, me, tgt, tmo, status = barrier
        arr = (C.c_void_p * len(flags))(*[ptr_of(f) for f in flags])
        n_m = len(flags)
    st = _lib.kv_switch_range(cache._h, ra.ptr, ra.n, gpu_lo, gpu_hi, arr, n_m, me, int(tgt), int(tmo),
                              ptr_of(status), stream_of(stream), C.byref(h))
    plan = Plan(cache, h, ra.n) if h.value else None
    if st != KV_OK:
        raise FlyKVError(st, _lib.kv_last_error().decode(), [plan] if plan is not None else [])
    return plan


def kv_switch_multi(cache: KVCache, waves, stream=None) -> list:
    """A switch in waves in one C call (kv_switch_multi): waves is a list of
    request lists (kv_plan_waves slices, or kv_plan_pieces waves through
    piece_request); no host sync between waves.  Returns one Plan per wave."""
    waves = [list(w) for w in waves]
    ra = make_requests([r for w in waves for r in w])
    ptr = np.zeros(len(waves) + 1, dtype=np.int32)
    np.cumsum([len(w) for w in waves], out=ptr[1:])
    hs = (C.c_void_p * max(len(waves), 1))()
    st = _lib.kv_switch_multi(cache._h, ra.ptr, ptr.ctypes.data_as(_I32P), len(waves), stream_of(stream), hs)
    plans = [Plan(cache, C.c_void_p(hs[k]), len(w)) if hs[k] else None for k, w in enumerate(waves)]
    if st != KV_OK:  # the waves before the failing one committed: hand them over
        raise FlyKVError(st, _lib.kv_last_error().decode(), [p for p in plans if p is not None])
    return plans


def kv_switch_waves(cache: KVCache, requests, max_wave_bytes: int = 0, split: bool = True, stream=None):
    """The whole memory-bounded switch in one C call (kv_switch_waves): the
    wave schedule (block-aligned token pieces with split, whole requests
    without) and every wave back to back, one sync.  Returns (waves, plans):
    waves[w] = [(request index, tok0, tok1)] in the order of plans[w]'s
    requests; a request's final table is the concatenation of its pieces'."""
    ra = make_requests(requests)
    cap = max(2 * ra.n, 16)
    while True:
        buf = (Piece * cap)()
        hs = (C.c_void_p * cap)()
        n_p, n_w = C.c_int32(), C.c_int32()
        st = _lib.kv_switch_waves(cache._h, ra.ptr, ra.n, int(max_wave_bytes), int(bool(split)), stream_of(stream),
                                  cap, buf, C.byref(n_p), hs, C.byref(n_w))
        if st == 1 and n_w.value == 0 and n_p.value > cap:  # INVALID_ARG with the needed count, nothing ran
            cap = n_p.value
            continue
        break
    plans = [Plan(cache, C.c_void_p(hs[k]), 0) if hs[k] else None for k in range(n_w.value)]
    waves = [[] for _ in range(n_w.value)]
    for k in range(min(n_p.value, cap)):
        pc = buf[k]
        if pc.wave < len(waves):
            waves[pc.wave].append((pc.req, pc.tok0, pc.tok1))
    for p, wv in zip(plans, waves):
        if p is not None:
            p.n_reqs = len(wv)
    if st != KV_OK:  # committed waves before the failing one: hand them (and their pieces) over
        err = FlyKVError(st, _lib.kv_last_error().decode(), [p for p in plans if p is not None])
        err.waves = [wv for p, wv in zip(plans, waves) if p is not None]
        raise err
    return waves, plans


def kv_switch_back(cache: KVCache, prev: Plan, stream=None) -> Plan:
    """kv_switch of the inverse of a committed plan (every request back to its
    source group), built inside the library."""
    h = C.c_void_p()
    st = _lib.kv_switch_back(cache._h, prev._h, stream_of(stream), C.byref(h))
    plan = Plan(cache, h, prev.n_reqs) if h.value else None
    if st != KV_OK:
        raise FlyKVError(st, _lib.kv_last_error().decode(), [plan] if plan is not None else [])
    return plan


def kv_suggest_rank_ids(cache: KVCache, requests, dst) -> list:
    """N2: movement-minimising rank-ID assignment of group dst's members."""
    ra = make_requests(requests)
    out = np.zeros(max(dst[1], 1), dtype=np.int32)
    _check(_lib.kv_suggest_rank_ids(cache._h, ra.ptr, ra.n, Group(*dst), out.ctypes.data_as(_I32P)))
    return [int(x) for x in out[:dst[1]]]


def kv_plan_waves(cache: KVCache, requests, max_wave_bytes: int = 0) -> list:
    """Memory-bounded waves: list of (start, end) request index ranges."""
    ra = make_requests(requests)
    arr, n = ra.ptr, ra.n
    ws = np.zeros(n + 2, dtype=np.int32)
    nw = C.c_int32()
    _check(_lib.kv_plan_waves(cache._h, arr, n, int(max_wave_bytes), ws.ctypes.data_as(_I32P), C.byref(nw)))
    return [(int(ws[k]), int(ws[k + 1])) for k in range(nw.value)]


def kv_plan_pieces(cache: KVCache, requests, max_wave_bytes: int = 0) -> list:
    """Memory-bounded waves that may split a request into block-aligned token
    pieces (R20): list of waves, each a list of (request index, tok0, tok1)."""
    ra = make_requests(requests)
    cap = max(2 * ra.n, 16)
    while True:
        buf = (Piece * cap)()
        n = C.c_int32()
        st = _lib.kv_plan_pieces(cache._h, ra.ptr, ra.n, int(max_wave_bytes), cap, buf, C.byref(n))
        if st == KV_OK:
            break
        if st == 1 and n.value > cap:  # INVALID_ARG with the needed count
            cap = n.value
            continue
        raise FlyKVError(st, _lib.kv_last_error().decode())
    waves = []
    for k in range(n.value):
        pc = buf[k]
        while len(waves) <= pc.wave:
            waves.append([])
        waves[pc.wave].append((pc.req, pc.tok0, pc.tok1))
    return waves


def piece_request(geom: Geometry, req, tok0: int, tok1: int):
    """The plain request that moves tokens [tok0, tok1) of `req` (a request
    tuple as for kv_plan_switch), for a piece from kv_plan_pieces: the
    library's kv_piece_request decides the source-table slice."""
    ra = make_requests([req])
    out = Request()
    _check(_lib.kv_piece_request(C.byref(geom), ra.ptr, int(tok0), int(tok1), C.byref(out)))
    base = ra.keep[0].__array_interface__["data"][0] if ra.keep else 0
    ptr = C.cast(out.src_blocks, C.c_void_p).value or 0
    first = (ptr - base) // 4 if ptr else 0
    ids = np.asarray(req[3], dtype=np.int32).reshape(-1)[first:first + out.n_src_blocks].copy()
    return (req[0], out.num_tokens, tuple(req[2]), ids, tuple(req[4])) + tuple(req[5:])


def kv_reshard(plan: Plan, gpu: int = -1, stream=None):
    _check(_lib.kv_reshard(plan._h, gpu, stream_of(stream)))


def kv_verify_replicas(plan: Plan, stream=None):
    """R10: (mismatching source atoms, first mismatch code or None) of the
    plan's replicated sources (synchronises the stream)."""
    n, first = C.c_int64(), C.c_uint64()
    _check(_lib.kv_verify_replicas(plan._h, stream_of(stream), C.byref(n), C.byref(first)))
    return n.value, (None if first.value == (1 << 64) - 1 else first.value)


def kv_reshard_range(plan: Plan, gpu_lo: int, gpu_hi: int, stream=None):
    """kv_reshard of the atoms sourced on pools [gpu_lo, gpu_hi), one launch."""
    _check(_lib.kv_reshard_range(plan._h, gpu_lo, gpu_hi, stream_of(stream)))


def kv_reshard_staged(plan: Plan, gpu: int, staging, staging_bytes: int, mode: int, stream=None):
    """Bench comparator: mode 1 pack -> staging, mode 2 unpack staging -> destinations."""
    _check(_lib.kv_reshard_staged(plan._h, gpu, ptr_of(staging), int(staging_bytes), mode, stream_of(stream)))


def a2a_offsets(plan: "Plan"):
    """(send_off, recv_off) for all_to_all_single buffers (kv_plan_a2a_offsets):
    send_off[s] = kv_pack's chunk_off for source s, recv_off[d] = kv_unpack's
    for destination d; int64 [n, n] byte offsets."""
    send, recv, _ = plan.a2a_offsets()
    return send, recv


def kv_pack(plan: Plan, src_gpu: int, buf, chunk_off, stream=None):
    """Gather src_gpu's atoms into per-destination chunks of buf (chunk_off[d] = byte offset)."""
    off = np.ascontiguousarray(np.asarray(chunk_off, dtype=np.int64))
    _check(_lib.kv_pack(plan._h, src_gpu, ptr_of(buf), off.ctypes.data_as(_I64P), stream_of(stream)))


def kv_unpack(plan: Plan, dst_gpu: int, buf, chunk_off, stream=None):
    """Scatter the chunks received by dst_gpu (chunk_off[s] = byte offset of s's chunk) into its pool."""
    off = np.ascontiguousarray(np.asarray(chunk_off, dtype=np.int64))
    _check(_lib.kv_unpack(plan._h, dst_gpu, ptr_of(buf), off.ctypes.data_as(_I64P), stream_of(stream)))


def kv_remap_block_tables(plan: Plan, gpu: int, req_ptr, block_ids, per_req_meta, stream=None):
    _check(_lib.kv_remap_block_tables(plan._h, gpu, ptr_of(req_ptr), ptr_of(block_ids), ptr_of(per_req_meta),
                                      stream_of(stream)))


# ----------------------------------------------------------------- weights
def weight_shard_view(desc: WeightDesc, rank: int, degree: int) -> View:
    v = View()
    _check(_lib.weight_shard_view(C.byref(desc), rank, degree, C.byref(v)))
    return v


def weight_desc(ptr, rows, cols, elem_bytes, kind, ld=None, num_q_heads=0, num_kv_heads=0, head_dim=0):
    return WeightDesc(ptr_of(ptr), rows, cols, cols if ld is None else ld, elem_bytes, kind, num_q_heads,
                      num_kv_heads, head_dim)


def kv_gather_view(view: View, dst, stream=None):
    _check(_lib.kv_gather_view(C.byref(view), ptr_of(dst), stream_of(stream)))


class VmmBuffer:
    """A weight buffer in CUDA VMM memory (kv_vmm_alloc): aliasable views."""

    def __init__(self, nbytes: int, device: int = 0):
        h, p = C.c_void_p(), C.c_void_p()
        _check(_lib.kv_vmm_alloc(device, nbytes, C.byref(h), C.byref(p)))
        self._h = h
        self.ptr = int(p.value)
        self.nbytes = nbytes

    def close(self):
        if getattr(self, "_h", None):
            _lib.kv_vmm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def vmm_granularity(device: int = 0) -> int:
    g = C.c_uint64()
    _check(_lib.kv_vmm_granularity(device, C.byref(g)))
    return g.value


def weight_view_alias(buf: VmmBuffer, view: View):
    """(contiguous device pointer, bytes) aliasing the view's segments."""
    p, n = C.c_void_p(), C.c_uint64()
    _check(_lib.weight_view_alias(buf._h, C.byref(view), C.byref(p), C.byref(n)))
    return int(p.value), n.value


def weight_view_unalias(ptr: int, nbytes: int):
    _check(_lib.weight_view_unalias(ptr, nbytes))


# ----------------------------------------------------------------- consumer proof
def kv_paged_decode(geom: Geometry, layer_base, n_res: int, req_ptr, block_ids, per_req_meta, seq_lens,
                    q_heads_local: int, q, out, scale: float, max_seq_len: int, stream=None, after_decode=False):
    """N3 paged decode attention over one layer of one pool (kv_paged_decode);
    max_seq_len >= every seq_lens entry (sizes the split workspace).
    after_decode: the previous kernel on the stream is a kv_paged_decode
    launch (KV_DECODE_AFTER_DECODE: the launches overlap)."""
    _check(_lib.kv_paged_decode(C.byref(geom), ptr_of(layer_base), n_res, ptr_of(req_ptr), ptr_of(block_ids),
                                ptr_of(per_req_meta), ptr_of(seq_lens), q_heads_local, ptr_of(q), ptr_of(out),
                                float(scale), int(max_seq_len), KV_DECODE_AFTER_DECODE if after_decode else 0,
                                stream_of(stream)))


def kv_paged_decode_release(stream=None):
    """Free the decode workspace kept for `stream` (kv_paged_decode_release)."""
    _check(_lib.kv_paged_decode_release(stream_of(stream)))


# ----------------------------------------------------------------- IPC
def ipc_export(dptr):
    h = (C.c_uint8 * 64)()
    off = C.c_uint64()
    _check(_lib.kv_ipc_export(ptr_of(dptr), h, C.byref(off)))
    return bytes(h), off.value


def ipc_import(handle: bytes, offset: int) -> int:
    h = (C.c_uint8 * 64).from_buffer_copy(handle)
    p = C.c_void_p()
    _check(_lib.kv_ipc_import(h, offset, C.byref(p)))
    return int(p.value)


def ipc_close(dptr: int, offset: int):
    _check(_lib.kv_ipc_close(dptr, offset))


def kv_group_barrier(flags, self_index: int, target: int, timeout_ns: int, status=None, stream=None):
    """Device-side group barrier (a5): flags = this process's pointers to
    every member's 64-bit counter; waits for counter[self] >= target."""
    arr = (C.c_void_p * len(flags))(*[ptr_of(f) for f in flags])
    _check(_lib.kv_group_barrier(arr, len(flags), self_index, int(target), int(timeout_ns), ptr_of(status),
                                 stream_of(stream)))


def group_barrier_selftest(n_members: int, rounds: int, absent: int = -1, timeout_ns: int = int(5e9)):
    """kv_group_barrier_selftest: the device barrier run by n_members members
    emulated as the CTAs of one cooperative launch.  Returns (errors,
    timeouts): ordering violations seen (must be 0) and members that ended
    their wait by timeout (those waiting on `absent`)."""
    e, t = C.c_int32(0), C.c_int32(0)
    _check(_lib.kv_group_barrier_selftest(n_members, rounds, absent, int(timeout_ns), C.byref(e), C.byref(t)))
    return int(e.value), int(t.value)


def stream_sync(stream=None):
    _check(_lib.kv_stream_sync(stream_of(stream)))


# ----------------------------------------------------------------- NVLS (N2)
class PoolMem:
    """One pool in a single shareable physical allocation (kv_pool_alloc /
    kv_pool_import): .ptr device address, .nbytes; tensor() views it."""

    def __init__(self, handle, ptr: int, nbytes: int, device: int):
        self._h = handle
        self.ptr = ptr
        self.nbytes = nbytes
        self.device = device

    @classmethod
    def alloc(cls, device: int, nbytes: int, align: int = 0) -> "PoolMem":
        h, p, n = C.c_void_p(), C.c_void_p(), C.c_uint64()
        _check(_lib.kv_pool_alloc(device, nbytes, align, C.byref(h), C.byref(p)))
        _check(_lib.kv_pool_size(h, C.byref(n)))
        return cls(h, int(p.value), int(n.value), device)

    @classmethod
    def import_fd(cls, fd: int, nbytes: int, device: int) -> "PoolMem":
        h, p = C.c_void_p(), C.c_void_p()
        _check(_lib.kv_pool_import(fd, nbytes, device, C.byref(h), C.byref(p)))
        return cls(h, int(p.value), nbytes, device)

    def export_fd(self) -> int:
        fd = C.c_int32()
        _check(_lib.kv_pool_export(self._h, C.byref(fd)))
        return fd.value

    def tensor(self, shape=None):
        """A torch uint8 tensor aliasing the pool (no copy); shape may cover
        less than the (granularity-rounded) allocation."""
        import torch

        class _Cai:
            def __init__(s, ptr, n):
                s.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False), "version": 3}
        t = torch.as_tensor(_Cai(self.ptr, self.nbytes), device=f"cuda:{self.device}")
        if shape is None:
            return t
        n = 1
        for x in shape:
            n *= x
        return t[:n].view(*shape)

    def free(self):
        if getattr(self, "_h", None):
            _lib.kv_pool_free(self._h)
            self._h = None


def mc_supported(n_devices: int, nbytes: int):
    """(ok, granularity, reason): can the driver create an NVLS multicast
    object for a team of n_devices (kv_mc_supported)?"""
    ok, g = C.c_int32(), C.c_uint64()
    st = _lib.kv_mc_supported(n_devices, nbytes, C.byref(ok), C.byref(g))
    return bool(ok.value), int(g.value), ("" if st == KV_OK else _lib.kv_last_error().decode())


class Multicast:
    """An NVLS multicast object of one replica team (kv_mc_*)."""

    def __init__(self, handle, fd: int = -1):
        self._h = handle
        self.fd = fd
        self.va = 0

    @classmethod
    def create(cls, n_devices: int, nbytes: int) -> "Multicast":
        h, fd = C.c_void_p(), C.c_int32()
        _check(_lib.kv_mc_create(n_devices, nbytes, C.byref(h), C.byref(fd)))
        return cls(h, fd.value)

    @property
    def nbytes(self) -> int:
        n = C.c_uint64()
        _check(_lib.kv_mc_size(self._h, C.byref(n)))
        return int(n.value)

    @classmethod
    def import_fd(cls, fd: int, nbytes: int, n_devices: int) -> "Multicast":
        h = C.c_void_p()
        _check(_lib.kv_mc_import(fd, nbytes, n_devices, C.byref(h)))
        return cls(h)

    def add_device(self, device: int):
        _check(_lib.kv_mc_add_device(self._h, device))

    def bind(self, pool: PoolMem):
        _check(_lib.kv_mc_bind(self._h, pool._h))

    def map(self, device: int) -> int:
        p = C.c_void_p()
        _check(_lib.kv_mc_map(self._h, device, C.byref(p)))
        self.va = int(p.value)
        return self.va

    def free(self):
        if getattr(self, "_h", None):
            _lib.kv_mc_free(self._h)
            self._h = None


def close_fd(fd: int):
    _lib.kv_close_fd(fd)
