"""flykv: B200-native KV Cache Adaptor re-layout (Flying Serving, arXiv 2602.22593).

The product path is libflykv.so (include/flykv.h): a C++ host planner and
sm_100a CUDA kernels.  ``flykv`` is its ctypes binding, ``pools`` allocates
paged pools with torch (device memory plumbing), ``comm`` holds the eagerly
built communicator pool and the peer-pool exchange for one process per GPU.
"""
from . import flykv  # noqa: F401  (raises if libflykv.so is missing)
from .flykv import (KVCache, Plan, kv_blocks_for, kv_gather_view, kv_layout, kv_plan_switch,  # noqa: F401
                    kv_remap_block_tables, kv_reshard, weight_shard_view)
