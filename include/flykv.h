/*
 * flykv.h -- C ABI of libflykv.so: the KV Cache Adaptor DP<->TP re-layout
 * and the zero-copy weight shard view of Flying Serving (arXiv 2602.22593),
 * built for NVIDIA B200 (sm_100a).
 *
 * Citations: P:n = line n of the paper's LaTeX, S:n = SPEC.md,
 * Rn = reading n in DESIGN.md section 3.
 *
 * Conventions for every entry point
 *   - Returns kv_status; KV_OK == 0.  No exceptions cross the ABI.  On error
 *     kv_last_error() returns a thread-local message with detail.
 *   - "host" pointers are CPU memory owned by the caller and only read (or
 *     written, for outputs) during the call.  "device" pointers are CUDA
 *     global memory owned by the caller; the library never frees them.
 *   - The library owns kv_cache and kv_plan objects (and their device
 *     workspaces); release them with kv_cache_destroy / kv_plan_destroy.
 *   - One caller thread per kv_cache.
 *   - Layout terms (R1-R4):
 *       L layers, H KV heads, d head_dim, B = B_base tokens per DP block,
 *       e bytes per element (2 for bf16);
 *       H_loc(p) = H/p if p <= H else 1                  (Eq.3, R2)
 *       B(p)     = B * H / H_loc(p)  (= p*B when p | H)   (Eq.2)
 *       M        = 2*H*B*d*e bytes per block per layer    (M_block P:338-340, R1)
 *     A block of one layer at degree p is [2 (K,V)][H_loc(p)][B(p)][d]
 *     elements, K first (R4; BJ north_star "[blocks, K/V, kv_heads,
 *     block_size, head_dim]").  Rank r of a degree-p group holds heads
 *     [r*H_loc, (r+1)*H_loc) (p <= H, R3) or head r/(p/H) (p > H, R2).
 */
#ifndef FLYKV_H
#define FLYKV_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KV_OK = 0,
    KV_ERR_INVALID_ARG = 1,        /* null pointer, negative size, bad geometry        */
    KV_ERR_INDIVISIBLE_DEGREE = 2, /* p does not divide H and H does not divide p (R2) */
    KV_ERR_UNKNOWN_GROUP = 3,      /* group not an aligned segment of a degree in {1} U P */
    KV_ERR_RANK_OUT_OF_RANGE = 4,  /* weight view rank outside [0, m)          */
    KV_ERR_INDIVISIBLE_EXTENT = 5, /* weight extent not divisible by m         */
    KV_ERR_OUT_OF_BLOCKS = 6,      /* destination does not fit; state unchanged */
    KV_ERR_BAD_BLOCK_TABLE = 7,    /* wrong length, out of range, not held, or shared (R14) */
    KV_ERR_DUPLICATE_REQUEST = 8,  /* same req_id twice in one plan (S:207 DoubleAllocate) */
    KV_ERR_BAD_STATE = 9,          /* call out of order (e.g. reshard after commit)    */
    KV_ERR_CUDA = 10,              /* a CUDA runtime call failed; see kv_last_error()  */
    KV_ERR_REPLICA_MISMATCH = 11,  /* strict mode: replicated source heads differ (R10) */
    KV_ERR_BARRIER = 12            /* a host barrier callback reported failure (kv_switch_range_host) */
} kv_status;

/* Model KV geometry.  block_base = B (DP tokens per block).  Requirement:
 * B*d*e (one "atom", the bytes of B tokens of one head) is a multiple of 16. */
typedef struct {
    int32_t num_layers;
    int32_t num_kv_heads;
    int32_t head_dim;
    int32_t block_base;
    int32_t elem_bytes;
} kv_geometry;

/* A DP engine (degree 1) or an aligned TP group [first_gpu, first_gpu+degree)
 * (only aligned contiguous segments; first_gpu % degree == 0). */
typedef struct {
    int32_t first_gpu;
    int32_t degree;
} kv_group;

/* One live request to re-lay-out.  src_blocks: host array of the request's
 * block IDs at the source degree, length n_src_blocks == ceil(num_tokens /
 * B(src.degree)) (uniform across the source group, R6).  Caller-owned.
 * src_rank_ids / dst_rank_ids (optional, NULL = identity, R3): host arrays
 * of degree entries, a permutation; member engine first_gpu + m of the group
 * holds the head slice of rank ID rank_ids[m] ("the Manager assigns each
 * engine a unique rank ID r"; the weight view of that engine is then
 * View(W, dim, rank_ids[m], degree), Eq.1).  kv_suggest_rank_ids picks a
 * movement-minimising assignment. */
typedef struct {
    int64_t req_id;
    int32_t num_tokens;
    kv_group src;
    const int32_t* src_blocks;
    int32_t n_src_blocks;
    kv_group dst;
    const int32_t* src_rank_ids;
    const int32_t* dst_rank_ids;
} kv_request;

typedef struct kv_cache kv_cache; /* opaque: pools, allocator bitmaps      */
typedef struct kv_plan kv_plan;   /* opaque: validated, allocated switch    */

/* Plan statistics (algorithmic bytes). */
typedef struct {
    int64_t n_requests;     /* requests in the plan                         */
    int64_t n_moving;       /* requests with src != dst                     */
    int64_t n_atoms;        /* source atoms read (B*d*e bytes each)         */
    int64_t n_atom_writes;  /* destination atoms written (>= n_atoms, GQA)  */
    int64_t atom_bytes;     /* B*d*e                                        */
    int64_t payload_bytes;  /* n_atom_writes * atom_bytes                   */
    int64_t h2d_bytes;      /* descriptor bytes uploaded per plan           */
    int64_t n_segments;     /* (request, source GPU) work segments          */
    int64_t n_atom_slots;   /* work slots of the kernels: one per atom plus
                               the mixed order's holes (>= n_atoms); the
                               staging size of kv_reshard_staged           */
    int64_t n_buckets;      /* destination buckets of the kernels' work
                               order, summed over source GPUs
                               (kv_cache_set_work_order)                    */
    /* host wall time of the phases of a kv_switch* call that ran this plan
     * (0 otherwise), for attributing switch latency (R15): */
    int64_t t_plan_ns;      /* kv_plan_switch: validate, allocate, plan     */
    int64_t t_enqueue_ns;   /* descriptor upload + reshard + remap enqueue  */
    int64_t t_wait_ns;      /* stream synchronisation: the device work      */
    int64_t t_read_ns;      /* copy of the tables into the plan             */
} kv_plan_stats;

/* ---------------------------------------------------------------- cache */

/*
 * kv_cache_create: register the per-GPU paged KV pools and the set of
 * supported TP degrees P (the paper's per-worker persistent pool P:223, the
 * fixed-M physical block pool P:334-340, aligned groups P:421-424).
 *   geom            host, layout geometry (validated; see kv_geometry)
 *   n_gpus          number of pools ("GPUs"/engines); several pools may live
 *                   on one physical device ("virtual ranks")
 *   num_blocks      host [n_gpus], blocks in each pool (same IDs in every layer, R5)
 *   layer_base      host [n_gpus * num_layers] device pointers, row-major by
 *                   GPU: layer l of GPU g starts at layer_base[g*L + l] and
 *                   holds num_blocks[g] * M bytes, 16-byte aligned.  The
 *                   pointers must be dereferenceable from the device that
 *                   later runs kv_reshard (local, same-device virtual ranks,
 *                   or peer/IPC-mapped over NVLink).  May be fake (never
 *                   dereferenced) if kv_reshard is never called.  The cache
 *                   binds to the device current at its first upload; device
 *                   calls made later from another device fail with
 *                   KV_ERR_BAD_STATE.
 *   tp_degrees      host [n_degrees], the set P (degree 1 is always legal)
 * All blocks start free.  No CUDA call is made here.
 */
kv_status kv_cache_create(const kv_geometry* geom, int32_t n_gpus, const int32_t* num_blocks,
                          void* const* layer_base, const int32_t* tp_degrees, int32_t n_degrees,
                          kv_cache** out);
/* Destroy a cache.  Plans of the cache that are still alive are detached:
 * their device workspaces and tables are released here (after their last
 * stream drains), and every later call on them returns KV_ERR_BAD_STATE
 * except kv_plan_destroy (which then frees the handle), kv_plan_get_stats
 * and kv_plan_dst_tables.  Destroy plans first to keep their tables. */
void kv_cache_destroy(kv_cache* cache);

/* Layout helpers (Eq.2/Eq.3): *h_loc = H_loc(p), *block_tokens = B(p),
 * *block_bytes = M.  KV_ERR_INDIVISIBLE_DEGREE if neither p | H nor H | p. */
kv_status kv_layout(const kv_geometry* geom, int32_t degree, int32_t* h_loc, int32_t* block_tokens,
                    int64_t* block_bytes);
/* *n = ceil(num_tokens / B(degree)) blocks per rank. */
kv_status kv_blocks_for(const kv_geometry* geom, int32_t num_tokens, int32_t degree, int32_t* n);

/* ------------------------------------------------------------ allocator */

/* kv_alloc: take the n lowest block IDs free on every GPU of group g and
 * mark them held on all members (Alg.1 "KVCacheMgr.Allocate" P:493; uniform
 * IDs R6, lowest-first R8).  out_ids: host [n].  OUT_OF_BLOCKS leaves the
 * state unchanged. */
kv_status kv_alloc(kv_cache* cache, kv_group g, int32_t n, int32_t* out_ids);
/* kv_reserve: mark the given IDs held on every GPU of g (registers a live
 * request whose table already exists).  BAD_BLOCK_TABLE if any ID is out of
 * range or already held; state unchanged on error. */
kv_status kv_reserve(kv_cache* cache, kv_group g, const int32_t* ids, int32_t n);
/* kv_free: release IDs on every GPU of g.  BAD_BLOCK_TABLE if any is
 * not held; state unchanged on error. */
kv_status kv_free(kv_cache* cache, kv_group g, const int32_t* ids, int32_t n);
/* *n_free = free blocks of pool gpu (conservation checks). */
kv_status kv_free_count(const kv_cache* cache, int32_t gpu, int32_t* n_free);
/* held: host [num_blocks[gpu]] bytes, 1 = held. */
kv_status kv_held_mask(const kv_cache* cache, int32_t gpu, uint8_t* held);

/* ---------------------------------------------------------------- switch */

/*
 * kv_plan_switch: validate and plan the re-layout of reqs[0..n_reqs) (host,
 * caller order = the globally agreed Q_wait order) and allocate every
 * destination table (a1-a3 of DESIGN.md section 1).
 *   For each request with src != dst: n1 = ceil(T / B(dst.degree)) IDs, the
 *   lowest free on every destination GPU, not taken earlier in this plan
 *   (R6, R8).  src == dst requests are no-ops that keep their table (R12).
 * Validation (state unchanged on any error):
 *   INVALID_ARG          null pointers, n_reqs < 0, num_tokens < 0
 *   UNKNOWN_GROUP        group not aligned / degree not in {1} U P / out of range
 *   INDIVISIBLE_DEGREE   degree incompatible with H (R2)
 *   BAD_BLOCK_TABLE      n_src_blocks != ceil(T/B(src)), ID out of range, ID not
 *                        held on every source GPU, or an ID in two requests (R14)
 *   DUPLICATE_REQUEST    req_id repeated
 *   OUT_OF_BLOCKS        destination does not fit next to the sources (R13)
 * The plan is a deterministic function of (cache state, reqs): every SPMD
 * process builds the identical plan.  No CUDA call is made here; descriptors
 * are uploaded to the device at the first kv_reshard.
 */
kv_status kv_plan_switch(kv_cache* cache, const kv_request* reqs, int32_t n_reqs, kv_plan** out);

/* kv_plan_upload: enqueue on `stream` the host->device copy of the plan's
 * descriptors (segments, tables, remap records: kv_plan_stats.h2d_bytes,
 * from pinned staging) into a stream-ordered device workspace.  Optional:
 * kv_reshard / kv_remap_block_tables upload on first use.  Lets a caller
 * prefetch descriptors while earlier work runs.  Idempotent. */
kv_status kv_plan_upload(kv_plan* plan, void* stream);

/*
 * kv_reshard: move the bytes (a4, the hot loop).  Enqueues on `stream`
 * (a cudaStream_t, NULL = legacy default) the copy of every atom whose
 * canonical source replica (R10) lives on pool `gpu`, or of all atoms when
 * gpu == -1 (all pools addressable from the current device, e.g. virtual
 * ranks on one B200).  An atom (request, layer, K/V, head, chunk of B
 * tokens) is B*d*e contiguous bytes in every degree's layout; it is read
 * once and written to each destination replica (1, or p/H under GQA
 * replication, R2), local or over NVLink peer mappings; inside a request
 * atoms are visited in destination-major order so destination blocks are
 * written sequentially, and across requests in the cache's work order
 * (kv_cache_set_work_order: mixed by default, so concurrent senders do not
 * converge on one receiver).  Idempotent until
 * the plan is committed.  The caller must order kv_remap_block_tables after
 * every GPU's reshard has completed (stream order, or a group barrier, a5).
 * Current device must be the one that can address the pools.
 */
kv_status kv_reshard(kv_plan* plan, int32_t gpu, void* stream);

/* kv_reshard_range: kv_reshard of the atoms sourced on pools [gpu_lo,
 * gpu_hi), one launch -- for a process that owns several pools (virtual
 * ranks) of a cache whose other pools belong to other processes.  kv_reshard
 * (gpu) == kv_reshard_range(gpu, gpu + 1); kv_reshard(-1) == range [0,
 * n_gpus).  A range short of every pool may store into peer mappings: the
 * kernel then ends with a system-scope fence for kv_group_barrier.
 * Errors: KV_ERR_INVALID_ARG (range empty or outside [0, n_gpus)),
 * KV_ERR_BAD_STATE (plan committed), KV_ERR_CUDA. */
kv_status kv_reshard_range(kv_plan* plan, int32_t gpu_lo, int32_t gpu_hi, void* stream);

/* Bench comparator only: the same re-layout split into two
 * passes through a staging buffer, as a pack -> all-to-all -> unpack
 * implementation would do.  mode 1 packs every atom of the range (source
 * replica) into staging[(i - first) * B*d*e]; mode 2 unpacks staging to
 * every destination replica.  staging: device, >= n_atom_slots * B*d*e bytes. */
kv_status kv_reshard_staged(kv_plan* plan, int32_t gpu, void* staging, int64_t staging_bytes, int32_t mode,
                            void* stream);

/*
 * The alternative cross-GPU path BJ names next to direct P2P stores: pack
 * into contiguous per-destination send buffers, an all-to-all (NCCL
 * all_to_all_single, by the caller), unpack (SURVEY 8(e) comparator N6).
 * Same bytes as kv_reshard; two extra HBM passes and a payload-sized buffer.
 *
 * Chunk (s -> d) holds every (atom, replica) sourced on GPU s whose
 * destination is GPU d, its size in bytes is bytes_matrix[s * n_gpus + d] of
 * kv_plan_get_stats.  Its layout: for each of s's segments (requests in plan
 * order), the atoms of the heads held by d's member of the destination group,
 * B*d*e bytes each, per (layer, K/V) by destination block, then head, then
 * chunk -- the order in which they fill d's blocks.  A function of the plan
 * alone, so every process derives it.
 *
 * kv_pack: enqueue on `stream` the gather of GPU src_gpu's atoms into chunks:
 *   buf        device, src_gpu's send buffer
 *   chunk_off  host int64 [n_gpus]: byte offset in buf of the chunk for
 *              each destination GPU (e.g. the exclusive prefix of row src_gpu
 *              of the bytes matrix for all_to_all_single)
 * kv_unpack: enqueue on `stream` the scatter of every chunk received by
 * dst_gpu into its pool's destination blocks:
 *   buf        device, dst_gpu's receive buffer
 *   chunk_off  host int64 [n_gpus]: byte offset in buf of the chunk from each
 *              source GPU (the exclusive prefix of column dst_gpu)
 * Both read the plan's uploaded descriptors; valid until the plan commits
 * (BAD_STATE after).  n_gpus <= 64.  The caller orders unpack after the
 * all-to-all, and the all-to-all after every pack.
 */
kv_status kv_pack(kv_plan* plan, int32_t src_gpu, void* buf, const int64_t* chunk_off, void* stream);
kv_status kv_unpack(kv_plan* plan, int32_t dst_gpu, const void* buf, const int64_t* chunk_off, void* stream);

/* Sizes of pool gpu's table after the switch: *n_resident requests resident
 * on gpu (dst group contains gpu), *n_ids block IDs in their tables; gpu ==
 * -1 gives the totals over all pools.  The per_req_meta first head of
 * kv_remap_block_tables follows the request's dst_rank_ids. */
kv_status kv_plan_resident(const kv_plan* plan, int32_t gpu, int32_t* n_resident, int32_t* n_ids);

/*
 * kv_remap_block_tables: a6 + a7.  Enqueues on `stream` a kernel writing
 * the post-switch "logical table" of pool gpu for the plan's
 * requests resident on it, in plan order:
 *   req_ptr       device int32 [n_resident + 1]  CSR row pointers
 *   block_ids     device int32 [n_ids]           destination block IDs
 *   per_req_meta  device int32 [4 * n_resident]  {plan request index, B(p),
 *                 H_loc(p), first head held by gpu} = the per-request
 *                 "stride and capacity" the attention kernel needs
 * gpu == -1 (all pools addressable from the current device): one launch
 * writes every pool's table into packed outputs, pool g's slice starting at
 * req_ptr + sum_{g'<g}(n_res[g'] + 1), block_ids + sum_{g'<g} n_ids[g'],
 * per_req_meta + 4 * sum_{g'<g} n_res[g'] (sizes from kv_plan_resident;
 * req_ptr then holds n_resident_total + n_gpus entries).
 * The first call on a plan (any gpu) commits it on the host: every moving
 * request's source IDs are released on its source GPUs (sources are freed
 * only after the group barrier, R13).  The released IDs can be handed out by
 * the very next kv_alloc / kv_plan_switch, so device work that writes them
 * (the next plan's reshard) must be ordered after this plan's reshard: the
 * same stream, or an event the caller records.  Requests absent from the
 * plan are not listed and are untouched.
 */
/* kv_plan_packed_offsets: where pool g's table starts in the packed outputs
 * of kv_remap_block_tables(gpu = -1), as element offsets: out host
 * [n_gpus * 3] = {req_ptr offset, block_ids offset, per_req_meta offset}
 * per pool (the prefix sums stated above); totals (element counts of the
 * three buffers) in totals host [3] or NULL.  Errors: INVALID_ARG, BAD_STATE. */
kv_status kv_plan_packed_offsets(const kv_plan* plan, int32_t* out, int64_t* totals);

kv_status kv_remap_block_tables(kv_plan* plan, int32_t gpu, int32_t* req_ptr, int32_t* block_ids,
                                int32_t* per_req_meta, void* stream);

/*
 * kv_switch: the whole switch in one call, for a process that addresses
 * every pool (virtual ranks, or peers mapped into one process):
 * kv_plan_switch -> descriptor upload -> kv_reshard(all pools) -> (stream
 * order is the barrier, a5) -> kv_remap_block_tables(all pools) into a
 * plan-owned device buffer -> one device->host copy of every pool's table ->
 * stream synchronisation.  On KV_OK the switch has completed, the plan is
 * committed (sources released, R13) and kv_plan_tables gives the tables on
 * the device (for the attention kernels) and on the host.  Errors from the
 * planner leave no state change and *out NULL; a CUDA error after the remap
 * returns the (committed) plan in *out so the caller can destroy it.
 * Switch latency (R15) is this call's wall time.  Not for one process per
 * GPU: there the group barrier sits between reshard and remap.
 */
kv_status kv_switch(kv_cache* cache, const kv_request* reqs, int32_t n_reqs, void* stream, kv_plan** out);

/* kv_switch_back: kv_switch of the inverse of a committed plan -- every
 * request from its destination (table, rank IDs) back to its source group
 * (the paper's reset_TP_mode after set_TP_mode), built inside the
 * library from the plan (no request list crosses the ABI).  The new plan
 * allocates fresh blocks like any switch.  BAD_STATE if prev is not
 * committed; INVALID_ARG if prev belongs to another cache. */
kv_status kv_switch_back(kv_cache* cache, const kv_plan* prev, void* stream, kv_plan** out);

/*
 * kv_switch_range: kv_switch for one process of a one-process-per-GPU job
 * that owns pools [gpu_lo, gpu_hi) (every process calls it with the same
 * request list): kv_plan_switch -> descriptor upload ->
 * kv_reshard_range(gpu_lo, gpu_hi) (pushes into peer pools) ->
 * kv_group_barrier(barrier_flags, n_members, self, barrier_target,
 * timeout_ns, barrier_status) when n_members > 1 (a5: every member's pushes
 * have landed) -> kv_remap_block_tables of each owned pool into the
 * plan-owned packed buffer -> one device->host copy -> stream sync.  On
 * KV_OK the owned pools' tables are available through kv_plan_tables (other
 * pools' slices are not written).  Barrier arguments as for
 * kv_group_barrier (the caller keeps the per-group counts).  Errors as
 * kv_switch; a barrier timeout is reported by *barrier_status (or a trap
 * when it is NULL), not by the return value.
 */
kv_status kv_switch_range(kv_cache* cache, const kv_request* reqs, int32_t n_reqs, int32_t gpu_lo, int32_t gpu_hi,
                          uint64_t* const* barrier_flags, int32_t n_members, int32_t self, uint64_t barrier_target,
                          int64_t timeout_ns, int32_t* barrier_status, void* stream, kv_plan** out);

/*
 * kv_switch_range_host: kv_switch_range with a HOST barrier in place of
 * kv_group_barrier (a5): after the owned pools' pushes the library
 * synchronizes `stream` (the push kernel ends with a system-scope fence, so
 * its peer stores are visible), then calls barrier(barrier_ctx) -- the
 * caller's host barrier over the members (e.g. a gloo / NCCL barrier);
 * when it returns every member's pushes have landed -- then remaps the
 * owned pools and reads the tables back as kv_switch_range does.  For
 * processes whose pools cannot spin on one another's device counters: ranks
 * that share one GPU (separate launches that wait on one another are not
 * guaranteed to be co-scheduled on one device), or peers without mapped
 * counters.  barrier NULL: no other process is involved.
 *   barrier  int32_t fn(void* ctx), returns 0 on success; called once, on the
 *            calling thread, with no library lock held
 * Errors as kv_switch_range; a non-zero callback return gives
 * KV_ERR_BARRIER and the (uncommitted) plan is rolled back.
 */
typedef int32_t (*kv_host_barrier_fn)(void* ctx);
kv_status kv_switch_range_host(kv_cache* cache, const kv_request* reqs, int32_t n_reqs, int32_t gpu_lo,
                               int32_t gpu_hi, kv_host_barrier_fn barrier, void* barrier_ctx, void* stream,
                               kv_plan** out);

/* kv_switch_multi: a switch in waves (kv_plan_waves, or the block-aligned
 * pieces of kv_plan_pieces turned into plain requests) with no host sync
 * between the waves: each wave is planned once the previous one committed
 * on the host, its kernels are stream-ordered after the previous wave's
 * (blocks a wave read may be the next wave's destinations), and the tables
 * of every wave are read back after one stream sync at the end.
 *   reqs      host, every wave's requests back to back
 *   wave_ptr  host [n_waves + 1], wave w = reqs[wave_ptr[w] .. wave_ptr[w+1])
 *   plans     host [n_waves] out: one committed plan per wave, tables as for
 *             kv_switch (kv_plan_tables); entries stay NULL past a failure,
 *             the caller destroys the non-NULL ones.
 * Errors: as kv_plan_switch / kv_switch for the failing wave.  The earlier
 * waves have committed (their sources are released) and completed, and
 * their tables have been read back: plans[0..w-1] are the caller's only
 * record of where those requests now live -- keep them.  plans[w] is set
 * if the failing wave committed before its error (its host tables are then
 * unavailable: kv_plan_tables(on_device = 0) returns BAD_STATE). */
kv_status kv_switch_multi(kv_cache* cache, const kv_request* reqs, const int32_t* wave_ptr, int32_t n_waves,
                          void* stream, kv_plan** plans);

/* kv_plan_tables: pool gpu's post-switch table of a plan run by kv_switch,
 * as pointers into plan-owned memory (valid until kv_plan_destroy):
 * on_device != 0 -> device pointers, else host pointers.  Layout as written
 * by kv_remap_block_tables (sizes from kv_plan_resident).  BAD_STATE if the
 * plan was not executed by kv_switch, or (host pointers) if its switch did
 * not complete the read-back. */
kv_status kv_plan_tables(const kv_plan* plan, int32_t gpu, int32_t on_device, const int32_t** req_ptr,
                         const int32_t** block_ids, const int32_t** per_req_meta);

/* kv_plan_commit: a7 on the host -- release every moving request's source
 * IDs (R13).  Implied by the first kv_remap_block_tables; call it directly
 * when the caller builds its block tables itself.  Idempotent.  Only after
 * every GPU's reshard of this plan has completed (group barrier). */
kv_status kv_plan_commit(kv_plan* plan);

/*
 * kv_plan_waves: memory-bounded waves (for the memory-driven
 * long-context promotion).  Partitions reqs (in order) into
 * consecutive waves such that each wave, planned after the previous waves
 * have been committed (their sources released), fits next to its own
 * sources, and (if max_wave_bytes > 0) moves at most max_wave_bytes of
 * destination payload unless a single request exceeds it.  Simulates the
 * allocator; no state change.  wave_start: host [n_reqs + 1], wave k is
 * reqs[wave_start[k] .. wave_start[k+1]); *n_waves >= 1 (0 for an empty list,
 * with only wave_start[0] = 0 written).  OUT_OF_BLOCKS if a
 * request does not fit even alone.  The caller then runs, per wave:
 * kv_plan_switch -> kv_reshard -> barrier -> kv_remap_block_tables.
 */
kv_status kv_plan_waves(const kv_cache* cache, const kv_request* reqs, int32_t n_reqs, int64_t max_wave_bytes,
                        int32_t* wave_start, int32_t* n_waves);

/*
 * kv_plan_pieces: memory-bounded waves that may split a request (R20): the
 * memory-driven promotion of ONE long request (Use Case 3)
 * when its source and destination do not fit side by side.  A request moves
 * in consecutive token pieces [tok0, tok1), each starting and (but for the
 * last) ending on a whole block of both layouts, so a piece is itself a
 * plain request: num_tokens = tok1 - tok0, src_blocks = the request's table
 * from tok0 / B(src degree) on, same groups and rank IDs.  Each wave is
 * planned after the previous waves committed (their pieces' source blocks
 * released); a piece takes the lowest common free IDs of its wave, and the
 * request's final table is the concatenation of its pieces' tables.  Whole
 * requests are kept whole when they fit (then this equals kv_plan_waves).
 *   pieces  host [cap] out: {wave, request index, tok0, tok1}, in wave order,
 *           request order within a wave; *n_pieces = count (also when cap is
 *           too small: INVALID_ARG, call again with that cap)
 * OUT_OF_BLOCKS if some piece cannot progress even in a wave of its own.
 * Simulates the allocator; no state change.
 */
typedef struct {
    int32_t wave, req, tok0, tok1;
} kv_piece;
kv_status kv_plan_pieces(const kv_cache* cache, const kv_request* reqs, int32_t n_reqs, int64_t max_wave_bytes,
                         int32_t cap, kv_piece* pieces, int32_t* n_pieces);

/* kv_piece_request: the plain request that moves tokens [tok0, tok1) of
 * *req (a piece of kv_plan_pieces, R20): num_tokens = tok1 - tok0,
 * src_blocks = req->src_blocks + tok0 / B(src degree) (a pointer into the
 * caller's table, not a copy), n_src_blocks = ceil(tok1 / B(src)) -
 * tok0 / B(src), same req_id, groups and rank IDs.  tok0 must start a
 * source block (tok0 % B(src) == 0, as every piece does) and 0 <= tok0 <
 * tok1 <= num_tokens; the whole range returns *req unchanged.  Errors:
 * INVALID_ARG (NULL pointers, range), INDIVISIBLE_DEGREE (src degree). */
kv_status kv_piece_request(const kv_geometry* geom, const kv_request* req, int32_t tok0, int32_t tok1,
                           kv_request* out);

/* kv_switch_waves: the whole memory-bounded switch in one call -- the wave
 * schedule (split = 0: kv_plan_waves, whole requests; split = 1:
 * kv_plan_pieces, block-aligned token pieces of a request when it cannot
 * move whole), each piece turned into a plain request, and kv_switch_multi.
 *   pieces    host [cap] out: the schedule {wave, request, tok0, tok1}
 *             (whole requests have tok0 = 0, tok1 = num_tokens); *n_pieces
 *   plans     host [cap] out: one committed plan per wave; *n_waves
 * A request's final table is the concatenation, in wave order, of the
 * destination tables of its pieces.  Errors: as kv_plan_waves /
 * kv_plan_pieces (INVALID_ARG with *n_pieces = the needed cap when cap is
 * too small; no state change) and kv_switch_multi. */
kv_status kv_switch_waves(kv_cache* cache, const kv_request* reqs, int32_t n_reqs, int64_t max_wave_bytes,
                          int32_t split, void* stream, int32_t cap, kv_piece* pieces, int32_t* n_pieces,
                          kv_plan** plans, int32_t* n_waves);

/* kv_suggest_rank_ids: N2 egress reduction.  For the requests of reqs whose
 * destination is group dst, choose the rank-ID assignment of dst's members
 * (out: host [dst.degree], rank ID of member m) that maximises the bytes
 * already resident on the engine that will own them (exact assignment over
 * the members, deterministic: ties keep the lower rank ID on the lower
 * member).  Pass it as dst_rank_ids of those requests.  No state change. */
kv_status kv_suggest_rank_ids(const kv_cache* cache, const kv_request* reqs, int32_t n_reqs, kv_group dst,
                              int32_t* out_rank_ids);

/* Host copies of every destination table, in plan order: dst_ptr host
 * [n_reqs+1], dst_ids host [dst_ptr[n_reqs]] (pass dst_ids = NULL to size). */
kv_status kv_plan_dst_tables(const kv_plan* plan, int32_t* dst_ptr, int32_t* dst_ids);
/* Statistics; bytes_matrix (host [n_gpus*n_gpus] or NULL) receives the
 * destination bytes each source GPU sends to each destination GPU (row =
 * source), the input of the roofline of SURVEY 8(d). */
kv_status kv_plan_get_stats(const kv_plan* plan, kv_plan_stats* stats, int64_t* bytes_matrix);

/* kv_plan_a2a_offsets: the byte offsets of kv_pack / kv_unpack for
 * all_to_all_single buffers, from the plan's bytes matrix (a function of
 * the plan alone, so every process derives the same):
 *   send_off  host [n_gpus * n_gpus] out (or NULL): send_off[s*n + d] =
 *             offset of chunk (s -> d) in s's send buffer = sum over d' < d
 *             of bytes[s][d'] (chunks in destination order)
 *   recv_off  host [n_gpus * n_gpus] out (or NULL): recv_off[d*n + s] =
 *             offset of chunk (s -> d) in d's receive buffer = sum over
 *             s' < s of bytes[s'][d] (chunks in source order)
 *   packed    host [n_gpus * n_gpus] out (or NULL): offset of chunk (s -> d)
 *             in ONE buffer holding every chunk in row-major (s, d) order
 *             (all pools in one process: pack then unpack in place)
 * Row s of send_off is kv_pack's chunk_off for src_gpu s; row d of recv_off
 * is kv_unpack's chunk_off for dst_gpu d.  Errors: INVALID_ARG, BAD_STATE. */
kv_status kv_plan_a2a_offsets(const kv_plan* plan, int64_t* send_off, int64_t* recv_off, int64_t* packed);
/* The kernel work order of source GPU `gpu` (kv_cache_set_work_order), for
 * link models: *n_rows receives the number of consecutive 1024-slot ranges of
 * the GPU's kernel slot order; out (host [n_rows * (n_gpus + 1)] or NULL)
 * receives, per range in visiting order, the destination bytes it writes to
 * each GPU (replicas included, holes excluded) and, in column n_gpus, the
 * bytes it reads on `gpu`.  Summed over ranges, the first n_gpus columns are
 * row `gpu` of kv_plan_get_stats' bytes_matrix.
 * Errors: KV_ERR_INVALID_ARG (NULL plan / n_rows, gpu out of range). */
kv_status kv_plan_work_order(const kv_plan* plan, int32_t gpu, int32_t* n_rows, int64_t* out);
/* Destroy a plan.  A plan that was never committed rolls back its
 * destination allocations.  Safe on a plan detached by kv_cache_destroy. */
void kv_plan_destroy(kv_plan* plan);

/* ------------------------------------------------------- weight views */

typedef enum {
    KV_W_COLUMN = 0,   /* column-parallel [out, in]: rank takes out-rows */
    KV_W_ROW = 1,      /* row-parallel [out, in]: rank takes in-columns  */
    KV_W_QKV = 2       /* fused stacked [Q; K; V] rows, head-aligned (R17, GQA R2)    */
} kv_weight_kind;

typedef struct {
    const void* ptr;      /* device (or host) base of the full matrix     */
    int64_t rows;         /* out features                                  */
    int64_t cols;         /* in features                                   */
    int64_t ld;           /* elements between consecutive rows (>= cols)  */
    int32_t elem_bytes;
    int32_t kind;         /* kv_weight_kind                                */
    int32_t num_q_heads;  /* KV_W_QKV only                                 */
    int32_t num_kv_heads; /* KV_W_QKV only                                 */
    int32_t head_dim;     /* KV_W_QKV only                                 */
} kv_weight_desc;

typedef struct {
    const void* ptr;  /* first element of the segment (inside the full matrix) */
    int64_t rows, cols, ld;
    int64_t row0, col0; /* position of the segment in the full matrix       */
} kv_view_segment;

typedef struct {
    int32_t n_seg;            /* 1 (COLUMN, ROW) or 3 (QKV: Q, K, V)          */
    int32_t elem_bytes;
    kv_view_segment seg[3];
} kv_view;

/*
 * weight_shard_view: Eq.1 W_active^(r) = View(W_full, dim, r, m).
 * Pure pointer arithmetic on the caller's matrix: 0 bytes moved or
 * allocated; the segments alias the full matrix.  rank in [0, m)
 * else RANK_OUT_OF_RANGE; the sharded extent must divide by m (QKV: Hq % m
 * and Hkv % m, or m % Hkv under GQA replication) else INDIVISIBLE_EXTENT.
 */
kv_status weight_shard_view(const kv_weight_desc* full, int32_t rank, int32_t degree, kv_view* out);

/* Contiguous zero-copy views ("contiguous in virtual memory but map
 * to the existing physical memory of the DP replica").  kv_vmm_alloc gives a
 * weight buffer backed by a CUDA VMM physical allocation (cuMemCreate,
 * size rounded up to the granularity, *dptr its device address);
 * weight_view_alias maps the view's row segments (COLUMN / QKV views, ld ==
 * cols) back to back into a fresh virtual range aliasing the same physical
 * memory: one contiguous [sum rows, cols] operand, 0 bytes copied.  Each
 * segment's offset and size must be multiples of kv_vmm_granularity
 * (INDIVISIBLE_EXTENT otherwise, e.g. Llama-3-70B QKV at TP2/4/8 fits);
 * strided ROW views are INVALID_ARG.  Writes through either address are
 * visible through the other.  weight_view_unalias releases the range. */
typedef struct kv_vmm_buffer kv_vmm_buffer;
kv_status kv_vmm_granularity(int32_t device, uint64_t* granularity);
kv_status kv_vmm_alloc(int32_t device, uint64_t bytes, kv_vmm_buffer** out, void** dptr);
kv_status kv_vmm_free(kv_vmm_buffer* buf);
kv_status weight_view_alias(const kv_vmm_buffer* buf, const kv_view* view, void** contiguous, uint64_t* bytes);
kv_status weight_view_unalias(void* contiguous, uint64_t bytes);

/* Test utility (DESIGN.md a8): gather a view's segments, in order, into the
 * contiguous device buffer dst (row-major, total rows x cols of the
 * segments) on `stream`.  Used only to check views against the oracle. */
kv_status kv_gather_view(const kv_view* view, void* dst, void* stream);

/* ------------------------------------------------------- consumer proof */

/*
 * kv_paged_decode: SURVEY 8(f) N3 -- paged decode attention over one layer
 * of one pool, reading the cache through the per-request "stride and
 * capacity" the Adaptor gives the attention kernel: the CSR table of
 * kv_remap_block_tables (req_ptr, block_ids) and per_req_meta {index, B(p),
 * H_loc(p), first KV head}.  Local query head j uses local KV head
 * j / (q_heads_local / H_loc) (GQA).  out[r][j] = softmax(scale * q.K^T) V
 * over tokens 0..seq_lens[r]-1 (zeros for seq_lens[r] = 0).  Tensor-core
 * flash decoding (mma.sync m16n8k16, bf16 in, fp32 accumulate, P as bf16
 * hi + lo), tiles of 16 tokens and splits of 512 tokens fixed in token
 * index, folded in a fixed order: a TP rank and the DP replica produce
 * identical bits for the same head.  HBM-bound: reads every K/V byte of the
 * resident requests once.
 *   layer_base  device, layer l region of the pool (16-byte aligned)
 *   block_ids   device; may be NULL when no resident request has a token
 *   q_heads_local  a multiple of every resident request's H_loc
 *   q           device bf16 [n_res][q_heads_local][head_dim] (16-byte aligned)
 *   out         device fp32 [n_res][q_heads_local][head_dim]
 *   max_seq_len host: >= every seq_lens entry; sizes the split workspace the
 *               library keeps per (device, stream) (a larger entry traps:
 *               a CUDA error, never a stray write)
 *   flags       0, or KV_DECODE_AFTER_DECODE: the kernel enqueued right
 *               before this one on the stream is a kv_paged_decode launch
 *               (e.g. the same layer of the next pool), or any kernel that
 *               does not let its dependents start early (no
 *               griddepcontrol.launch_dependents /
 *               cudaTriggerProgrammaticLaunchCompletion before it is done).
 *               The launch then overlaps a previous decode launch through
 *               programmatic dependent launch: it reads the cache, q and the
 *               tables before that launch completes (a decode grid never
 *               writes them) and waits only before its workspace and out.
 *               Wrong after a kernel that triggers its dependents early and
 *               writes q, the cache or the tables; without the flag a launch
 *               waits for the previous kernel as usual.  Other bits:
 *               KV_ERR_INVALID_ARG.
 * Calls on one stream share that workspace (ordered); calls on different
 * streams use different ones.  It grows outside stream capture only: a
 * call captured into a CUDA graph that would need a larger workspace
 * returns KV_ERR_BAD_STATE (call once with the same sizes before capturing).  bf16 and head_dim 64/128/256 only
 * (INVALID_ARG otherwise); KV_ERR_CUDA on workspace allocation or launch.
 */
#define KV_DECODE_AFTER_DECODE 1
kv_status kv_paged_decode(const kv_geometry* geom, const void* layer_base, int32_t n_res, const int32_t* req_ptr,
                          const int32_t* block_ids, const int32_t* per_req_meta, const int32_t* seq_lens,
                          int32_t q_heads_local, const void* q, float* out, float scale, int32_t max_seq_len,
                          int32_t flags, void* stream);

/* kv_paged_decode_release: free the decode workspace the library keeps for
 * `stream` on the current device (stream-ordered; a later kv_paged_decode on
 * that stream allocates a new one).  Call before destroying a stream that
 * ran kv_paged_decode.  KV_OK if there is none; KV_ERR_CUDA on failure. */
kv_status kv_paged_decode_release(void* stream);

/* ------------------------------------------------------- multi-process */

/* CUDA IPC helpers for peer pools (one process per GPU).  kv_ipc_export
 * writes a 64-byte handle of the allocation containing dptr plus dptr's
 * offset inside it; kv_ipc_import maps it (lazy peer access) in this
 * process and returns the base + offset pointer; kv_ipc_close unmaps
 * (pass the pointer kv_ipc_import returned). */
kv_status kv_ipc_export(const void* dptr, uint8_t handle[64], uint64_t* offset);
kv_status kv_ipc_import(const uint8_t handle[64], uint64_t offset, void** dptr);
kv_status kv_ipc_close(void* dptr, uint64_t offset);

/*
 * kv_group_barrier: the group completion barrier between processes (a5;
 * P:451 "safe points"), on the device, no host round trip.  Enqueues on
 * `stream` one single-thread kernel that (1) fences at system scope (every
 * earlier kernel of the stream -- this process's reshard and its NVLink
 * peer stores -- is ordered before what follows), (2) adds 1 with
 * system-scope release semantics to the 64-bit counter of every member,
 * then (3) spins with acquire loads on its own counter until it is
 * >= target.  Later work on the stream (the remap, the next switch) starts
 * only after every member's arrival, so after every member's pushes.
 *   flags       host array [n_members] of device pointers: this process's
 *               mapping of each member's counter (its own, or a peer's
 *               through kv_ipc_import); 8-byte aligned, zero-initialised
 *               once by its owner; one counter per (process, group)
 *   self        index of this process's own counter in flags
 *   target      k * n_members for the k-th barrier (k = 1, 2, ...) on
 *               these counters -- every member adds exactly once per
 *               barrier, so the count is exact and no reset is needed
 *   timeout_ns  a member that never arrives ends the wait after this long:
 *               *status (device int32, may be NULL) is set to 1; with
 *               status NULL the kernel traps (a CUDA error, never a hang)
 * Counters are caller memory; ranks outside the group do not call.
 * Errors: KV_ERR_INVALID_ARG (NULL / unaligned pointer, n_members outside
 * [1, 64], self out of range, timeout <= 0), KV_ERR_CUDA (launch).
 */
kv_status kv_group_barrier(uint64_t* const* flags, int32_t n_members, int32_t self, uint64_t target,
                           int64_t timeout_ns, int32_t* status, void* stream);

/*
 * kv_group_barrier_selftest (test utility): the device barrier of
 * kv_group_barrier run by n_members emulated members, the CTAs of ONE
 * cooperative launch on the current device (co-resident by construction;
 * separate launches that spin on one another must not share a device).
 * Per round k (1..rounds) member m stores k into its payload word, runs the
 * same arrive/wait code as flykv_barrier_kernel on counters laid out as for
 * kv_group_barrier (target k * n_members), then loads every member's
 * payload.  *errors = loads that saw a value < k (a member passed the
 * barrier before another's prior store was visible: must be 0); member
 * `absent` (-1: none) never arrives, so the others end their wait after
 * timeout_ns and *timeouts counts them.  Synchronous; allocates and frees
 * its own device memory.  Errors: KV_ERR_INVALID_ARG (n_members outside
 * [1, 64], rounds < 1, absent >= n_members, timeout <= 0, NULL outputs),
 * KV_ERR_CUDA.
 */
kv_status kv_group_barrier_selftest(int32_t n_members, int32_t rounds, int32_t absent, int64_t timeout_ns,
                                    int32_t* errors, int32_t* timeouts);

/* Make all prior writes of this device (incl. NVLink peer stores) visible
 * system-wide before a host-side barrier: synchronizes `stream`. */
kv_status kv_stream_sync(void* stream);

/* ------------------------------------------- NVLS multicast (N2, GQA) */
/*
 * GQA head replication (Eq.3): at a destination degree p > H,
 * head h lives on the aligned team of p/H engines [g0 + h*p/H, +p/H) at the
 * same block IDs and offsets.  With the team's pools bound to one NVLS
 * multicast object, a sender that is a member of the team writes each atom
 * once (multimem.st) and NVSwitch delivers it to every replica: its NVLink
 * egress is one copy instead of p/H.
 *
 * Pool memory for this path: one physical allocation per pool, POSIX-fd
 * shareable (kv_pool_alloc), mapped by peers through the exported descriptor
 * (kv_pool_export -> pass the fd, e.g. SCM_RIGHTS -> kv_pool_import) rather
 * than CUDA IPC.  align: round the size up to a multiple of this (the
 * multicast granularity from kv_mc_supported; 0 = allocation granularity).
 * The fd of kv_pool_export / kv_mc_create is the caller's (kv_close_fd).
 *
 * Team setup (every member process, in this order): the team leader
 * kv_mc_create(team size, pool bytes) and sends its fd; the others
 * kv_mc_import; every member kv_mc_add_device(own device); (all members
 * added) kv_mc_bind(own pool); (all bound) kv_mc_map -> the multicast VA;
 * then kv_cache_set_multicast(cache, team, layer bases inside that VA).
 * kv_mc_supported(n_devices, bytes): *ok = 1 if the driver creates a
 * multicast object of that team size (released again), else KV_ERR_CUDA
 * with the driver's reason; *granularity = the recommended granularity.
 * All: KV_ERR_INVALID_ARG on bad arguments, KV_ERR_CUDA with the driver's
 * error otherwise.
 */
typedef struct kv_pool_mem kv_pool_mem;
typedef struct kv_mc kv_mc;
kv_status kv_pool_alloc(int32_t device, uint64_t bytes, uint64_t align, kv_pool_mem** out, void** dptr);
kv_status kv_pool_export(const kv_pool_mem* pool, int32_t* fd);
kv_status kv_pool_import(int32_t fd, uint64_t bytes, int32_t device, kv_pool_mem** out, void** dptr);
kv_status kv_pool_free(kv_pool_mem* pool);
kv_status kv_mc_supported(int32_t n_devices, uint64_t bytes, int32_t* ok, uint64_t* granularity);
kv_status kv_mc_create(int32_t n_devices, uint64_t bytes, kv_mc** out, int32_t* fd);
kv_status kv_mc_import(int32_t fd, uint64_t bytes, int32_t n_devices, kv_mc** out);
kv_status kv_mc_add_device(kv_mc* mc, int32_t device);
kv_status kv_mc_bind(kv_mc* mc, const kv_pool_mem* pool);
kv_status kv_mc_map(kv_mc* mc, int32_t device, void** va);
kv_status kv_mc_free(kv_mc* mc);
kv_status kv_close_fd(int32_t fd);
/* Allocated sizes (rounded up to the granularity): what kv_pool_import /
 * kv_mc_import must be given on the other side. */
kv_status kv_pool_size(const kv_pool_mem* pool, uint64_t* bytes);
kv_status kv_mc_size(const kv_mc* mc, uint64_t* bytes);

/*
 * kv_cache_set_multicast: register the multicast mapping of replica team
 * `team` (first_gpu = its first pool, degree = its size r = p/H) for this
 * process: layer_base host [L] device pointers, layer l's region of every
 * member pool as seen through the multicast VA (same offsets as the
 * members' own layer_base).  From then on kv_reshard / kv_reshard_range
 * write every atom whose replicas are exactly this team (destination degree
 * p with p/H == r, identity destination rank IDs, replica 0 on first_gpu)
 * with one multimem.st per 16 bytes instead of r stores.  Register only
 * teams this process is a member of (a multicast VA is usable on member
 * devices only); other teams keep per-replica stores.  layer_base NULL
 * clears the team.  mode: 1 = multimem (the product path); 2 = emulation
 * for single-GPU tests -- layer_base are ordinary pointers and the kernel
 * stores once with st.global there (replicas 1..r-1 are NOT written), which
 * checks the addressing without NVLS hardware.  Takes effect for launches
 * after the call.  Errors: INVALID_ARG (team not aligned or r < 2, bad
 * mode), KV_ERR_CUDA (upload).
 */
kv_status kv_cache_set_multicast(kv_cache* cache, kv_group team, void* const* layer_base, int32_t mode);

/* ---------------------------------------------------------------- misc */
const char* kv_strerror(kv_status s);
const char* kv_last_error(void);
/*
 * kv_cache_set_work_order: the order in which each source GPU's kernel visits
 * its atoms in plans built from now on (results are identical either way:
 * every (atom, replica) is written once, to its own bytes).
 *   order 1 (default) mixed: the GPU's work is bucketed by destination
 *           group and the kernel walks it in quanta of about 1024 atom
 *           slots, each quantum taking its share (1/K) of every bucket, in an
 *           order rotated by the source GPU.  At every moment a sender's
 *           traffic is split over its receivers in the proportions of the
 *           whole switch, the assumption behind t_min.  When
 *           all GPUs push at once (one process per GPU, NVSwitch),
 *           concurrent senders therefore do not converge on one receiver --
 *           e.g. TP8 -> 8 x DP1, where every sender holds a slice of every
 *           request, no longer pushes request i from all 8 GPUs into engine
 *           i mod 8 at the same time (ingress hot-spot).
 *   order 0 plan order: each GPU's segments in request order.
 * Errors: KV_ERR_INVALID_ARG (NULL cache, order not 0/1).  DESIGN.md 8.
 */
kv_status kv_cache_set_work_order(kv_cache* cache, int32_t order);

/*
 * Strict replica mode (R10).  A source group of degree p0 > H holds each
 * head on p0/H ranks (Eq.3 replication); the re-layout reads the
 * lowest-owner replica only (canonical source, R10), so a corrupted replica
 * would go unnoticed -- or a corrupted canonical one would be propagated.
 *
 * kv_verify_replicas: enqueue on `stream` a kernel comparing, for every
 * moving request of the plan with p0 > H, every valid token (t < T) of
 * every layer, K/V half and head in each non-canonical replica with the
 * canonical replica; then one device->host copy and a stream sync.
 *   mismatches  host out: atoms (request, layer, K/V, head, B-token chunk,
 *               replica) with at least one differing valid byte
 *   first       host out (may be NULL): the smallest mismatch code,
 *               ((item * 2L + 2l + kv) << 32) | chunk, item = position in
 *               (request, head, replica >= 1) order; UINT64_MAX if none
 * Pools must be addressable from the current device.  Tail slots past T in
 * the last chunk are not compared (stale, R9).  Errors: INVALID_ARG,
 * BAD_STATE (committed or detached plan), KV_ERR_CUDA.
 *
 * kv_cache_set_strict(cache, 1): kv_switch / kv_switch_multi /
 * kv_switch_waves / kv_switch_back / kv_switch_range / kv_switch_range_host
 * verify every plan first (after its upload, before its reshard) and, on a
 * mismatch, roll the plan back (no state change, no byte moved) and return
 * KV_ERR_REPLICA_MISMATCH.  In a one-process-per-GPU job every process
 * checks every replicated item (peers' pools through their mappings), so
 * all processes reach the same decision.  Costs one read of every
 * replicated source byte and a host sync per plan with replicated sources.
 * Default 0 (off).
 */
kv_status kv_verify_replicas(kv_plan* plan, void* stream, int64_t* mismatches, uint64_t* first);
kv_status kv_cache_set_strict(kv_cache* cache, int32_t strict);

/* Tuning knob for the reshard kernel (process-wide): impl 0 = default
 * (LDG/STG warp copy, two atoms in flight per warp for 2/4 KiB atoms; for
 * >= 8 GQA replicas into local pools, the TMA bulk-copy ring with
 * lane-parallel replica stores), 1 = LDG/STG one atom per warp iteration,
 * 2 = TMA bulk-copy ring for every launch (local pools and kv_pack's send
 * chunks only; peer pools and NVLS teams always use LDG/STG), 3 = LDG/STG
 * with two atoms in flight, also for >= 8 replicas; ctas_per_sm 0 =
 * occupancy maximum.  Measured alternatives, see DESIGN.md section 7. */
kv_status kv_set_reshard_impl(int32_t impl, int32_t ctas_per_sm);

/* Number of kernels this library launched since load (evidence counter). */
int64_t kv_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FLYKV_H */
