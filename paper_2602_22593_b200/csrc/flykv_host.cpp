// flykv_host.cpp -- host side of libflykv.so: the C ABI declared in
// include/flykv.h, the block allocator (per-GPU bitmaps), the switch planner
// and the launches of the sm_100a kernels in flykv_kernels.cu.
//
// Citations: P:n = PAPER.md line, S:n = SPEC.md line, Rn = DESIGN.md reading.
#include "flykv.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <map>
#include <new>
#include <string>
#include <unordered_set>
#include <vector>

#include "flykv_internal.h"

using namespace flykv;

// ------------------------------------------------------------ errors
static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

static kv_status vfail(kv_status s, const char* fmt, va_list ap) {
    char buf[512];
    vsnprintf(buf, sizeof buf, fmt, ap);
    g_err = buf;
    return s;
}

static kv_status fail(kv_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vfail(s, fmt, ap);
    va_end(ap);
    return s;
}

// shared with flykv_vmm.cpp
kv_status flykv_fail(kv_status s, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vfail(s, fmt, ap);
    va_end(ap);
    return s;
}

static kv_status cuda_fail(cudaError_t e, const char* what) {
    return fail(KV_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CUDA_TRY(call)                                            \
    do {                                                          \
        cudaError_t _e = (call);                                  \
        if (_e != cudaSuccess) return cuda_fail(_e, #call);       \
    } while (0)

// ------------------------------------------------------------ objects
struct kv_cache {
    kv_geometry geo;
    int32_t n_gpus = 0;
    std::vector<int32_t> num_blocks;
    std::vector<void*> layer_base;        // [n_gpus * L]
    std::vector<int32_t> degrees;         // the set P (degree 1 always legal)
    std::vector<std::vector<uint64_t>> held;  // per GPU bitmap, bit = held
    int64_t M = 0;                        // block bytes per layer
    int64_t atom_bytes = 0;               // B*d*e
    // device copy of layer_base (uploaded once per device)
    int dev = -1;
    char** d_layer_base = nullptr;
    // stream-ordered pool for plan workspaces; keeps its memory across
    // synchronizations (release threshold = max) so a switch never waits on
    // the driver re-mapping freed workspace memory
    cudaMemPool_t pool = nullptr;
    // pinned staging for descriptor uploads: a ring of kStageRing buffers,
    // each guarded by an event, so planning wave w+1 never waits for the
    // upload of wave w (queued behind wave w-1's kernels) to be consumed
    static constexpr int kStageRing = 4;
    void* stage[kStageRing] = {};
    size_t stage_bytes[kStageRing] = {};
    cudaEvent_t stage_ev[kStageRing] = {};
    bool stage_pending[kStageRing] = {};
    int stage_next = 0;
    // plans not yet destroyed: kv_cache_destroy detaches them
    std::unordered_set<kv_plan*> live;
    // host table buffers of destroyed plans, reused by the next read-backs
    // (a fresh allocation of a few hundred KB page-faults on every switch)
    std::vector<std::vector<int32_t>> spare_h;
    // pinned landing buffer of kv_switch's one device->host table copy
    void* back = nullptr;
    size_t back_bytes = 0;
    // kernel work order of new plans: 1 = destination-rotated (default), 0 = plan order
    int32_t work_order = 1;
    // strict replica mode (kv_cache_set_strict, R10)
    int32_t strict = 0;
    // NVLS multicast teams of this process (kv_cache_set_multicast, N2):
    // mc_team[g] = size of the team whose first pool is g (0 = none),
    // mc_base[g*L + l] its layer-l multicast address; device copies uploaded
    // before the next reshard when dirty
    std::vector<int32_t> mc_team;
    std::vector<void*> mc_base;
    int32_t mc_mode = 0;
    bool mc_dirty = false;
    char** d_mc_base = nullptr;
    int32_t* d_mc_team = nullptr;
};

struct ReqPlan {
    int64_t req_id;
    int32_t T;
    kv_group src, dst;
    int32_t src_off, n0;  // source table in plan->tables
    int32_t dst_off, n1;  // destination table in plan->tables
    bool moving;
    int32_t src_rid[64], dst_rid[64];  // rank ID of each member, identity by default
    bool dst_rid_identity;
};

enum { PLAN_PLANNED = 0, PLAN_COMMITTED = 1 };

// A plan whose cache was destroyed (p->c == nullptr): every call but
// kv_plan_destroy / kv_plan_get_stats / kv_plan_dst_tables returns BAD_STATE.
#define PLAN_CHECK(p)                                                                         \
    do {                                                                                      \
        if (!(p)) return fail(KV_ERR_INVALID_ARG, "plan is NULL");                             \
        if (!(p)->c) return fail(KV_ERR_BAD_STATE, "the plan's cache was destroyed");          \
    } while (0)

struct kv_plan {
    kv_cache* c = nullptr;
    int state = PLAN_PLANNED;
    std::vector<ReqPlan> reqs;
    std::vector<int32_t> tables;
    std::vector<Seg> segs;
    // kernel work order (build_work_order).  Piece space: each source GPU's
    // segments, bucket after bucket; seg_begin is the exclusive prefix of
    // their slot counts, gpu_seg_lo/hi each GPU's range of positions
    std::vector<int32_t> seg_of;     // segment at each piece-space position
    std::vector<int64_t> seg_begin;
    std::vector<int32_t> gpu_seg_lo, gpu_seg_hi;
    std::vector<MixStream> streams;  // per source GPU: its mixed slot space
    std::vector<MixBucket> buckets;
    int64_t mixed_end = 0;           // slots of every GPU's mixed space (the kernels' atom index)
    std::vector<int64_t> bytes;  // n_gpus * n_gpus
    std::vector<int32_t> n_res, n_res_ids;
    std::vector<ReqRec> recs;
    kv_plan_stats st{};
    std::vector<int32_t> out_off;  // [n_gpus][3] packed all-GPU remap output offsets
    // pack -> all-to-all -> unpack (kv_pack / kv_unpack): per (segment, member)
    // atom base inside the chunk (source GPU -> member's GPU), and each
    // receiver's (segment, member) pairs
    std::vector<int64_t> a2a_base;
    std::vector<A2AItem> items;
    std::vector<int32_t> item_lo, item_hi;
    std::vector<int64_t> recv_atoms;
    // device workspace: [seg_begin | seg_of | streams | buckets | segs | tables | recs | out_off | a2a_base | items]
    int dev = -1;
    char* dbuf = nullptr;
    size_t dbytes = 0;
    size_t off_seg_begin = 0, off_seg_of = 0, off_streams = 0, off_buckets = 0, off_segs = 0, off_tables = 0, off_recs = 0, off_outs = 0, off_a2a = 0, off_items = 0;
    cudaStream_t last_stream = nullptr;
    // kv_switch: packed all-pool tables [req_ptr | block_ids | meta] on the
    // device (plan-owned, from the cache's pool) and their host copy
    int32_t* d_out = nullptr;
    std::vector<int32_t> h_out;
    int64_t out_rp = 0, out_ids = 0;  // element offsets of block_ids and meta in the packed buffer
};

// ------------------------------------------------------------ helpers
static inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

static kv_status check_geometry(const kv_geometry* g) {
    if (!g) return fail(KV_ERR_INVALID_ARG, "geometry is NULL");
    if (g->num_layers < 1 || g->num_kv_heads < 1 || g->head_dim < 1 || g->block_base < 1 ||
        g->elem_bytes < 1)
        return fail(KV_ERR_INVALID_ARG, "geometry fields must be >= 1");
    int64_t atom = (int64_t)g->block_base * g->head_dim * g->elem_bytes;
    if (atom % 16)
        return fail(KV_ERR_INVALID_ARG, "B*d*e = %lld bytes is not a multiple of 16", (long long)atom);
    int64_t M = 2 * (int64_t)g->num_kv_heads * atom;
    if (M > ((int64_t)1 << 40)) return fail(KV_ERR_INVALID_ARG, "block too large");
    return KV_OK;
}

// Degree compatibility with H (R2): p | H, or H | p (GQA replication).
static kv_status check_degree(int32_t H, int32_t p) {
    if (p < 1) return fail(KV_ERR_UNKNOWN_GROUP, "degree %d < 1", p);
    if (p <= H ? (H % p) : (p % H))
        return fail(KV_ERR_INDIVISIBLE_DEGREE, "degree %d incompatible with %d KV heads", p, H);
    return KV_OK;
}

// Aligned contiguous segment of a supported degree (R12).
static kv_status check_group(const kv_cache* c, kv_group g) {
    if (g.degree < 1 || g.degree > 64) return fail(KV_ERR_UNKNOWN_GROUP, "degree %d outside [1, 64]", g.degree);
    if (g.degree != 1 &&
        std::find(c->degrees.begin(), c->degrees.end(), g.degree) == c->degrees.end())
        return fail(KV_ERR_UNKNOWN_GROUP, "degree %d not in the pool's TP degrees", g.degree);
    if (g.first_gpu < 0 || g.first_gpu % g.degree || g.first_gpu + g.degree > c->n_gpus)
        return fail(KV_ERR_UNKNOWN_GROUP, "group [%d, +%d) is not an aligned segment of %d GPUs",
                    g.first_gpu, g.degree, c->n_gpus);
    return check_degree(c->geo.num_kv_heads, g.degree);
}

static inline bool bit_get(const std::vector<uint64_t>& bm, int32_t b) {
    return (bm[(size_t)b >> 6] >> (b & 63)) & 1u;
}
static inline void bit_set(std::vector<uint64_t>& bm, int32_t b) { bm[(size_t)b >> 6] |= 1ull << (b & 63); }
static inline void bit_clr(std::vector<uint64_t>& bm, int32_t b) { bm[(size_t)b >> 6] &= ~(1ull << (b & 63)); }

static int32_t group_min_blocks(const kv_cache* c, kv_group g) {
    int32_t nb = c->num_blocks[g.first_gpu];
    for (int32_t r = 1; r < g.degree; ++r) nb = std::min(nb, c->num_blocks[g.first_gpu + r]);
    return nb;
}

// The n lowest IDs free on every GPU of g (R6, R8): OR the members' held
// words, then walk free bits with count-trailing-zeros.  Marks them held on
// every member when found.  Returns false (nothing marked) if fewer than n.
typedef std::vector<std::vector<uint64_t>> Bitmaps;

// start_word (optional, in/out): the scan starts at this word, and on
// success it is advanced to the word of the last ID taken -- every ID below
// it is then held on the group (lowest-first), so a later allocation on the
// same group in the same plan can skip that prefix (allocations only add
// held bits until the plan commits).  The taken bits are set word-wise.
static bool alloc_lowest_in(const kv_cache* c, Bitmaps& held, kv_group g, int32_t n, int32_t* out,
                            int32_t* start_word = nullptr) {
    if (n == 0) return true;
    const int32_t nb = group_min_blocks(c, g);
    const int32_t words = (nb + 63) >> 6;
    int32_t got = 0, w = start_word ? *start_word : 0, w_first = w, w_last = w;
    thread_local std::vector<uint64_t> taken;
    taken.clear();
    for (; w < words && got < n; ++w) {
        uint64_t used = 0;
        for (int32_t r = 0; r < g.degree; ++r) used |= held[g.first_gpu + r][w];
        uint64_t fr = ~used;
        const int32_t top = nb - (w << 6);
        if (top < 64) fr &= (top <= 0) ? 0ull : ((1ull << top) - 1);
        uint64_t mask = 0;
        while (fr && got < n) {
            const uint64_t bit = fr & (~fr + 1);
            out[got++] = (w << 6) + __builtin_ctzll(fr);
            mask |= bit;
            fr ^= bit;
        }
        taken.push_back(mask);
        w_last = w;
    }
    if (got < n) return false;
    for (int32_t r = 0; r < g.degree; ++r) {
        std::vector<uint64_t>& bm = held[g.first_gpu + r];
        for (int32_t k = w_first; k <= w_last; ++k) bm[k] |= taken[k - w_first];
    }
    if (start_word) *start_word = w_last;
    return true;
}

static bool alloc_lowest(kv_cache* c, kv_group g, int32_t n, int32_t* out) {
    return alloc_lowest_in(c, c->held, g, n, out);
}

// ------------------------------------------------------------ cache API
extern "C" kv_status kv_cache_create(const kv_geometry* geom, int32_t n_gpus, const int32_t* num_blocks,
                                     void* const* layer_base, const int32_t* tp_degrees, int32_t n_degrees,
                                     kv_cache** out) {
    if (!out) return fail(KV_ERR_INVALID_ARG, "out is NULL");
    *out = nullptr;
    kv_status s = check_geometry(geom);
    if (s) return s;
    if (n_gpus < 1 || !num_blocks || !layer_base || n_degrees < 0 || (n_degrees > 0 && !tp_degrees))
        return fail(KV_ERR_INVALID_ARG, "bad pool arguments");
    const int32_t L = geom->num_layers;
    for (int32_t g = 0; g < n_gpus; ++g) {
        if (num_blocks[g] < 0) return fail(KV_ERR_INVALID_ARG, "num_blocks[%d] < 0", g);
        for (int32_t l = 0; l < L; ++l)
            if ((uintptr_t)layer_base[(size_t)g * L + l] & 15)
                return fail(KV_ERR_INVALID_ARG, "layer_base[%d][%d] not 16-byte aligned", g, l);
    }
    for (int32_t i = 0; i < n_degrees; ++i) {
        s = check_degree(geom->num_kv_heads, tp_degrees[i]);
        if (s) return s;
    }
    kv_cache* c = new (std::nothrow) kv_cache();
    if (!c) return fail(KV_ERR_INVALID_ARG, "out of host memory");
    c->geo = *geom;
    c->n_gpus = n_gpus;
    c->num_blocks.assign(num_blocks, num_blocks + n_gpus);
    c->layer_base.assign(layer_base, layer_base + (size_t)n_gpus * L);
    c->degrees.assign(tp_degrees, tp_degrees + n_degrees);
    c->held.resize(n_gpus);
    for (int32_t g = 0; g < n_gpus; ++g) c->held[g].assign(((size_t)num_blocks[g] + 63) / 64, 0ull);
    c->atom_bytes = (int64_t)geom->block_base * geom->head_dim * geom->elem_bytes;
    c->M = 2 * (int64_t)geom->num_kv_heads * c->atom_bytes;
    *out = c;
    return KV_OK;
}

extern "C" void kv_cache_destroy(kv_cache* c) {
    if (!c) return;
    // detach live plans: release their device workspaces (from this cache's
    // pool) now; the caller still owns the handles, and kv_plan_destroy on a
    // detached plan only frees its host memory
    for (kv_plan* p : c->live) {
        if (p->dbuf) cudaFreeAsync(p->dbuf, p->last_stream);
        if (p->d_out) cudaFreeAsync(p->d_out, p->last_stream);
        if (p->dbuf || p->d_out) cudaStreamSynchronize(p->last_stream);
        p->dbuf = nullptr;
        p->d_out = nullptr;
        p->c = nullptr;
    }
    c->live.clear();
    for (int k = 0; k < kv_cache::kStageRing; ++k) {
        if (c->stage_ev[k]) {
            cudaEventSynchronize(c->stage_ev[k]);
            cudaEventDestroy(c->stage_ev[k]);
        }
        if (c->stage[k]) cudaFreeHost(c->stage[k]);
    }
    if (c->back) cudaFreeHost(c->back);
    if (c->d_layer_base) cudaFree(c->d_layer_base);
    if (c->d_mc_base) cudaFree(c->d_mc_base);
    if (c->d_mc_team) cudaFree(c->d_mc_team);
    if (c->pool) cudaMemPoolDestroy(c->pool);
    delete c;
}

extern "C" kv_status kv_layout(const kv_geometry* geom, int32_t degree, int32_t* h_loc, int32_t* block_tokens,
                               int64_t* block_bytes) {
    kv_status s = check_geometry(geom);
    if (s) return s;
    s = check_degree(geom->num_kv_heads, degree);
    if (s) return s;
    Layout L = layout_of(geom->num_kv_heads, degree);
    if (h_loc) *h_loc = L.hloc;
    if (block_tokens) *block_tokens = geom->block_base * L.k;
    if (block_bytes)
        *block_bytes = 2 * (int64_t)geom->num_kv_heads * geom->block_base * geom->head_dim * geom->elem_bytes;
    return KV_OK;
}

extern "C" kv_status kv_blocks_for(const kv_geometry* geom, int32_t num_tokens, int32_t degree, int32_t* n) {
    int32_t bt = 0;
    kv_status s = kv_layout(geom, degree, nullptr, &bt, nullptr);
    if (s) return s;
    if (num_tokens < 0 || !n) return fail(KV_ERR_INVALID_ARG, "num_tokens < 0 or n NULL");
    *n = (int32_t)ceil_div(num_tokens, bt);
    return KV_OK;
}

// ------------------------------------------------------------ allocator API
extern "C" kv_status kv_alloc(kv_cache* c, kv_group g, int32_t n, int32_t* out_ids) {
    if (!c || n < 0 || (n > 0 && !out_ids)) return fail(KV_ERR_INVALID_ARG, "bad kv_alloc arguments");
    kv_status s = check_group(c, g);
    if (s) return s;
    if (!alloc_lowest(c, g, n, out_ids))
        return fail(KV_ERR_OUT_OF_BLOCKS, "%d blocks not free on group [%d,+%d)", n, g.first_gpu, g.degree);
    return KV_OK;
}

static kv_status check_ids(const kv_cache* c, kv_group g, const int32_t* ids, int32_t n, bool want_held) {
    const int32_t nb = group_min_blocks(c, g);
    std::vector<uint64_t> seen(((size_t)nb + 63) / 64, 0ull);
    for (int32_t k = 0; k < n; ++k) {
        const int32_t b = ids[k];
        if (b < 0 || b >= nb) return fail(KV_ERR_BAD_BLOCK_TABLE, "block id %d out of range", b);
        if (bit_get(seen, b)) return fail(KV_ERR_BAD_BLOCK_TABLE, "block id %d repeated", b);
        bit_set(seen, b);
        for (int32_t r = 0; r < g.degree; ++r)
            if (bit_get(c->held[g.first_gpu + r], b) != want_held)
                return fail(KV_ERR_BAD_BLOCK_TABLE, "block id %d is %s on GPU %d", b,
                            want_held ? "not held" : "already held", g.first_gpu + r);
    }
    return KV_OK;
}

extern "C" kv_status kv_reserve(kv_cache* c, kv_group g, const int32_t* ids, int32_t n) {
    if (!c || n < 0 || (n > 0 && !ids)) return fail(KV_ERR_INVALID_ARG, "bad kv_reserve arguments");
    kv_status s = check_group(c, g);
    if (s) return s;
    s = check_ids(c, g, ids, n, false);
    if (s) return s;
    for (int32_t r = 0; r < g.degree; ++r)
        for (int32_t k = 0; k < n; ++k) bit_set(c->held[g.first_gpu + r], ids[k]);
    return KV_OK;
}

extern "C" kv_status kv_free(kv_cache* c, kv_group g, const int32_t* ids, int32_t n) {
    if (!c || n < 0 || (n > 0 && !ids)) return fail(KV_ERR_INVALID_ARG, "bad kv_free arguments");
    kv_status s = check_group(c, g);
    if (s) return s;
    s = check_ids(c, g, ids, n, true);
    if (s) return s;
    for (int32_t r = 0; r < g.degree; ++r)
        for (int32_t k = 0; k < n; ++k) bit_clr(c->held[g.first_gpu + r], ids[k]);
    return KV_OK;
}

extern "C" kv_status kv_free_count(const kv_cache* c, int32_t gpu, int32_t* n_free) {
    if (!c || !n_free || gpu < 0 || gpu >= c->n_gpus) return fail(KV_ERR_INVALID_ARG, "bad arguments");
    int64_t held = 0;
    for (uint64_t w : c->held[gpu]) held += __builtin_popcountll(w);
    *n_free = (int32_t)(c->num_blocks[gpu] - held);
    return KV_OK;
}

extern "C" kv_status kv_held_mask(const kv_cache* c, int32_t gpu, uint8_t* held) {
    if (!c || !held || gpu < 0 || gpu >= c->n_gpus) return fail(KV_ERR_INVALID_ARG, "bad arguments");
    for (int32_t b = 0; b < c->num_blocks[gpu]; ++b) held[b] = bit_get(c->held[gpu], b) ? 1 : 0;
    return KV_OK;
}

// A request moves unless it stays in the same group with the same rank IDs (R12).
static bool request_moves(const kv_request& r) {
    if (r.src.first_gpu != r.dst.first_gpu || r.src.degree != r.dst.degree) return true;
    for (int32_t m = 0; m < r.src.degree; ++m) {
        const int32_t a = r.src_rank_ids ? r.src_rank_ids[m] : m;
        const int32_t b = r.dst_rank_ids ? r.dst_rank_ids[m] : m;
        if (a != b) return true;
    }
    return false;
}

// ------------------------------------------------------------ planner
// a2: validate a request list against the cache (no state change).
static kv_status validate_requests(const kv_cache* c, const kv_request* reqs, int32_t n_reqs, int64_t* total_src_out,
                                   int64_t* total_dst_bound_out) {
    const int32_t H = c->geo.num_kv_heads, B = c->geo.block_base;
    const int32_t n = c->n_gpus;
    std::unordered_set<int64_t> ids_seen;
    std::vector<std::vector<uint64_t>> in_plan(n);
    for (int32_t g = 0; g < n; ++g) in_plan[g].assign(c->held[g].size(), 0ull);
    int64_t total_src = 0, total_dst_bound = 0;
    for (int32_t i = 0; i < n_reqs; ++i) {
        const kv_request& r = reqs[i];
        if (r.num_tokens < 0) return fail(KV_ERR_INVALID_ARG, "request %d: num_tokens < 0", i);
        kv_status s = check_group(c, r.src);
        if (s) return s;
        s = check_group(c, r.dst);
        if (s) return s;
        if (!ids_seen.insert(r.req_id).second)
            return fail(KV_ERR_DUPLICATE_REQUEST, "req_id %lld repeated", (long long)r.req_id);
        for (int side = 0; side < 2; ++side) {
            const int32_t* rid = side ? r.dst_rank_ids : r.src_rank_ids;
            const int32_t p = side ? r.dst.degree : r.src.degree;
            if (!rid) continue;
            uint64_t seen = 0;
            for (int32_t m = 0; m < p; ++m) {
                if (rid[m] < 0 || rid[m] >= p || ((seen >> rid[m]) & 1ull))
                    return fail(KV_ERR_INVALID_ARG, "request %d: %s rank IDs are not a permutation of [0,%d)", i,
                                side ? "dst" : "src", p);
                seen |= 1ull << rid[m];
            }
        }
        const Layout l0 = layout_of(H, r.src.degree);
        const int64_t n0 = ceil_div(r.num_tokens, (int64_t)B * l0.k);
        if (r.n_src_blocks != n0 || (n0 > 0 && !r.src_blocks))
            return fail(KV_ERR_BAD_BLOCK_TABLE, "request %d: %d source blocks, expected %lld", i,
                        r.n_src_blocks, (long long)n0);
        const int32_t nb = group_min_blocks(c, r.src);
        for (int32_t k = 0; k < r.n_src_blocks; ++k) {
            const int32_t b = r.src_blocks[k];
            if (b < 0 || b >= nb) return fail(KV_ERR_BAD_BLOCK_TABLE, "request %d: block %d out of range", i, b);
            for (int32_t q = 0; q < r.src.degree; ++q) {
                const int32_t g = r.src.first_gpu + q;
                if (!bit_get(c->held[g], b))
                    return fail(KV_ERR_BAD_BLOCK_TABLE, "request %d: block %d not held on GPU %d", i, b, g);
                if (bit_get(in_plan[g], b))
                    return fail(KV_ERR_BAD_BLOCK_TABLE, "block %d of GPU %d appears twice in the plan (R14)", b, g);
                bit_set(in_plan[g], b);
            }
        }
        total_src += r.n_src_blocks;
        total_dst_bound += ceil_div(r.num_tokens, B);
    }

    *total_src_out = total_src;
    *total_dst_bound_out = total_dst_bound;
    return KV_OK;
}

// ---- kv_plan_switch, step by step ----

// Release the destination allocations of requests [0, upto) of a plan that
// will not run (failed planning, or destroyed before committing): S:207.
static void rollback_allocations(kv_plan* p, int32_t upto) {
    kv_cache* c = p->c;
    for (int32_t j = 0; j < upto; ++j) {
        const ReqPlan& u = p->reqs[j];
        if (!u.moving) continue;
        for (int32_t r = 0; r < u.dst.degree; ++r)
            for (int32_t k = 0; k < u.n1; ++k) bit_clr(c->held[u.dst.first_gpu + r], p->tables[u.dst_off + k]);
    }
}

// Per-request records and source tables (a2): rank IDs (identity unless
// given), and whether the request moves (R12/R19).
static void init_requests(kv_plan* p, const kv_request* reqs, int32_t n_reqs) {
    for (int32_t i = 0; i < n_reqs; ++i) {
        const kv_request& r = reqs[i];
        ReqPlan& q = p->reqs[i];
        q.req_id = r.req_id;
        q.T = r.num_tokens;
        q.src = r.src;
        q.dst = r.dst;
        for (int32_t m = 0; m < 64; ++m) {
            q.src_rid[m] = (r.src_rank_ids && m < r.src.degree) ? r.src_rank_ids[m] : m;
            q.dst_rid[m] = (r.dst_rank_ids && m < r.dst.degree) ? r.dst_rank_ids[m] : m;
        }
        q.dst_rid_identity = true;
        for (int32_t m = 0; m < r.dst.degree; ++m) q.dst_rid_identity &= q.dst_rid[m] == m;
        q.moving = request_moves(r);
        q.src_off = (int32_t)p->tables.size();
        q.n0 = r.n_src_blocks;
        p->tables.insert(p->tables.end(), r.src_blocks, r.src_blocks + r.n_src_blocks);
    }
}

// a3: destination tables in request order, lowest common free IDs (R6, R8);
// a no-op keeps its table (R12).  Returns the first request that does not
// fit (its predecessors' allocations are still held), or -1.
static int32_t allocate_destinations(kv_plan* p) {
    kv_cache* c = p->c;
    const int32_t H = c->geo.num_kv_heads, B = c->geo.block_base;
    std::vector<std::pair<int64_t, int32_t>> cursor;  // (group key, first word worth scanning)
    for (int32_t i = 0; i < (int32_t)p->reqs.size(); ++i) {
        ReqPlan& q = p->reqs[i];
        q.dst_off = (int32_t)p->tables.size();
        if (!q.moving) {
            q.n1 = q.n0;
            for (int32_t k = 0; k < q.n0; ++k) p->tables.push_back(p->tables[q.src_off + k]);
            continue;
        }
        const Layout l1 = layout_of(H, q.dst.degree);
        q.n1 = (int32_t)ceil_div(q.T, (int64_t)B * l1.k);
        p->tables.resize(p->tables.size() + q.n1);
        const int64_t key = ((int64_t)q.dst.first_gpu << 32) | (uint32_t)q.dst.degree;
        auto it = std::find_if(cursor.begin(), cursor.end(), [&](const auto& e) { return e.first == key; });
        if (it == cursor.end()) it = cursor.insert(cursor.end(), {key, 0});
        if (!alloc_lowest_in(c, c->held, q.dst, q.n1, p->tables.data() + q.dst_off, &it->second)) return i;
    }
    return -1;
}

// Rank-ID tables of non-identity destinations: rank ID of member m
// (remap's first head) and member of rank ID (reshard's owner lookup).
static void rank_id_tables(kv_plan* p, std::vector<int32_t>& rid_off, std::vector<int32_t>& inv_off) {
    const int32_t n_reqs = (int32_t)p->reqs.size();
    rid_off.assign(n_reqs, -1);
    inv_off.assign(n_reqs, -1);
    for (int32_t i = 0; i < n_reqs; ++i) {
        const ReqPlan& q = p->reqs[i];
        if (q.dst_rid_identity) continue;
        rid_off[i] = (int32_t)p->tables.size();
        p->tables.insert(p->tables.end(), q.dst_rid, q.dst_rid + q.dst.degree);
        inv_off[i] = (int32_t)p->tables.size();
        p->tables.resize(p->tables.size() + q.dst.degree);
        for (int32_t m = 0; m < q.dst.degree; ++m) p->tables[inv_off[i] + q.dst_rid[m]] = m;
    }
}

// Work segments (request, canonical source replica R10), the per-(source,
// destination) byte matrix, grouped by source GPU (stable: request order
// within a GPU).  seg_req: the request of each segment.  Returns the first
// request whose atom count overflows the device's 32-bit per-segment slot
// index, or -1.
static int32_t build_segments(kv_plan* p, const std::vector<int32_t>& inv_off, std::vector<Seg>& segs,
                              std::vector<int32_t>& seg_req) {
    const kv_cache* c = p->c;
    const int32_t H = c->geo.num_kv_heads, L = c->geo.num_layers, B = c->geo.block_base, n = c->n_gpus;
    p->bytes.assign((size_t)n * n, 0);
    for (int32_t i = 0; i < (int32_t)p->reqs.size(); ++i) {
        const ReqPlan& q = p->reqs[i];
        if (!q.moving) continue;
        const int32_t C = (int32_t)ceil_div(q.T, B);
        if (C == 0) continue;
        if ((int64_t)L * 2 * (C + H) * H >= ((int64_t)1 << 31)) return i;
        const Layout l0 = layout_of(H, q.src.degree), l1 = layout_of(H, q.dst.degree);
        int32_t inv1[64];
        for (int32_t m = 0; m < q.dst.degree; ++m) inv1[q.dst_rid[m]] = m;
        for (int32_t m = 0; m < q.src.degree; ++m) {
            const int32_t rid = q.src_rid[m];         // member m holds rank ID rid's slice
            if (l0.rep > 1 && rid % l0.rep) continue;  // only replica 0 of each head is read (R10)
            Seg sg{};
            sg.src_gpu = q.src.first_gpu + m;
            sg.dst_g0 = q.dst.first_gpu;
            sg.C = C;
            sg.J1 = (int32_t)ceil_div(C, l1.k);
            sg.nh = l0.hloc;
            sg.h0 = first_head_of_rank(l0, rid);
            sg.dst_inv = inv_off[i];
            sg.src_tab = q.src_off;
            sg.dst_tab = q.dst_off;
            sg.hloc0 = l0.hloc;
            sg.k0 = l0.k;
            sg.hloc1 = l1.hloc;
            sg.k1 = l1.k;
            sg.rep1 = l1.rep;
            segs.push_back(sg);
            seg_req.push_back(i);
            const int64_t head_bytes = (int64_t)L * 2 * C * c->atom_bytes;
            for (int32_t hh = 0; hh < sg.nh; ++hh)
                for (int32_t j = 0; j < l1.rep; ++j) {
                    const int32_t dg = sg.dst_g0 + inv1[owner_rank(l1, sg.h0 + hh, j)];
                    p->bytes[(size_t)sg.src_gpu * n + dg] += head_bytes;
                }
        }
    }
    std::vector<int32_t> order(segs.size());
    for (size_t k = 0; k < order.size(); ++k) order[k] = (int32_t)k;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) { return segs[a].src_gpu < segs[b].src_gpu; });
    std::vector<Seg> s2(segs.size());
    std::vector<int32_t> r2(segs.size());
    for (size_t k = 0; k < order.size(); ++k) {
        s2[k] = segs[order[k]];
        r2[k] = seg_req[order[k]];
    }
    segs.swap(s2);
    seg_req.swap(r2);
    return -1;
}

// Pack -> all-to-all -> unpack layout (kv_pack / kv_unpack).  Chunk (s -> d)
// = for each segment sourced on s (plan order), for the member m of its
// destination group on d: the atoms of the heads m holds (rank ID
// dst_rid[m]) in destination-major order (a2a_pos in flykv_kernels.cu).
static void build_a2a_layout(kv_plan* p, std::vector<Seg>& segs, const std::vector<int32_t>& seg_req) {
    const int32_t L = p->c->geo.num_layers, n = p->c->n_gpus;
    std::vector<int64_t> run((size_t)n * n, 0), tot(n, 0);
    std::vector<std::vector<A2AItem>> per(n);
    for (size_t k = 0; k < segs.size(); ++k) {
        Seg& sg = segs[k];
        const ReqPlan& q = p->reqs[seg_req[k]];
        sg.a2a = (int32_t)p->a2a_base.size();
        const int64_t per_head = (int64_t)L * 2 * sg.C;
        for (int32_t m = 0; m < q.dst.degree; ++m) {
            const int32_t rid = q.dst_rid[m];
            int32_t nh_m;
            if (sg.rep1 == 1) {
                const int32_t lo = std::max(sg.h0, rid * sg.hloc1), hi = std::min(sg.h0 + sg.nh, (rid + 1) * sg.hloc1);
                nh_m = std::max(0, hi - lo);
            } else {
                const int32_t h = rid / sg.rep1;
                nh_m = (h >= sg.h0 && h < sg.h0 + sg.nh) ? 1 : 0;
            }
            const int32_t d = sg.dst_g0 + m;
            int64_t& r = run[(size_t)sg.src_gpu * n + d];
            p->a2a_base.push_back(r);
            const int64_t cnt = nh_m * per_head;
            r += cnt;
            if (cnt > 0) {
                per[d].push_back(A2AItem{(int32_t)k, m, rid, nh_m, tot[d]});
                tot[d] += cnt;
            }
        }
    }
    p->item_lo.assign(n, 0);
    p->item_hi.assign(n, 0);
    p->recv_atoms = tot;
    for (int32_t d = 0; d < n; ++d) {
        p->item_lo[d] = (int32_t)p->items.size();
        p->items.insert(p->items.end(), per[d].begin(), per[d].end());
        p->item_hi[d] = (int32_t)p->items.size();
    }
}

// Kernel work order of each source GPU.  The GPU's segments
// are bucketed by destination group (order 1, the default) and laid out
// bucket after bucket (piece space); the kernel then walks a mixed slot space of
// K quanta, each quantum taking the next u_b = ceil(s_b / K) slots of every
// bucket b (s_b its slots; slots past s_b are holes), so at every moment a
// sender's traffic is split over its receivers in the proportions of the
// whole switch -- the assumption under t_min.  Without it, a
// TP group splitting into DP engines (TP8 -> 8 x DP1: every sender holds a
// slice of every request) pushes request i from all senders into engine
// i mod n at the same time (ingress hot-spot).  Buckets are
// visited in an order rotated by the source GPU.  Order 0: one bucket (plan
// order), K = 1.  Results do not depend on the order: every (atom, replica)
// is written once, to its own bytes.
static constexpr int64_t kQuantumSlots = 1024;  // target slots per quantum (4 MiB of 4 KiB atoms)

static void build_work_order(kv_plan* p, const std::vector<int64_t>& slots) {
    const int32_t n = p->c->n_gpus, H = p->c->geo.num_kv_heads;
    const std::vector<Seg>& segs = p->segs;
    p->seg_of.clear();
    p->seg_begin.clear();
    p->streams.assign(n, MixStream{});
    p->buckets.clear();
    p->gpu_seg_lo.assign(n, 0);
    p->gpu_seg_hi.assign(n, 0);
    int64_t acc = 0, mixed = 0;
    size_t k = 0;
    for (int32_t g = 0; g < n; ++g) {
        p->gpu_seg_lo[g] = (int32_t)p->seg_of.size();
        const size_t lo = k;
        while (k < segs.size() && segs[k].src_gpu == g) ++k;
        const size_t hi = k;
        // buckets: (rotated destination rank, destination degree) -> the GPU's segments, plan order
        std::vector<std::pair<int64_t, std::vector<int32_t>>> bk;
        for (size_t s = lo; s < hi; ++s) {
            const Seg& sg = segs[s];
            int64_t key = 0;
            if (p->c->work_order == 1)
                key = (int64_t)(((sg.dst_g0 - g) % n + n) % n) * 128 + (int64_t)(H / sg.hloc1) * sg.rep1;
            auto it = std::find_if(bk.begin(), bk.end(), [&](const auto& b) { return b.first == key; });
            if (it == bk.end()) bk.push_back({key, {(int32_t)s}});
            else it->second.push_back((int32_t)s);
        }
        std::stable_sort(bk.begin(), bk.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        MixStream& ms = p->streams[g];
        ms.begin = mixed;
        ms.b0 = (int32_t)p->buckets.size();
        ms.nb = (int32_t)bk.size();
        int64_t total = 0;
        for (const auto& b : bk) {
            MixBucket mb{};
            mb.start = acc;
            for (int32_t s : b.second) {
                p->seg_of.push_back(s);
                p->seg_begin.push_back(acc);
                acc += slots[s];
            }
            mb.size = acc - mb.start;
            total += mb.size;
            p->buckets.push_back(mb);
        }
        const int64_t K = bk.size() <= 1 ? 1 : std::max<int64_t>(1, total / kQuantumSlots);
        int64_t qs = 0;
        for (int32_t b = ms.b0; b < ms.b0 + ms.nb; ++b) {
            MixBucket& mb = p->buckets[b];
            mb.u = (int32_t)ceil_div(mb.size, K);
            mb.P = (int32_t)qs;
            qs += mb.u;
        }
        ms.Qs = (int32_t)std::max<int64_t>(qs, 1);
        ms.K = (int32_t)K;
        mixed += total ? K * qs : 0;
        p->gpu_seg_hi[g] = (int32_t)p->seg_of.size();
    }
    p->seg_begin.push_back(acc);
    p->mixed_end = mixed;
    p->st.n_buckets = (int64_t)p->buckets.size();
}

// The kernels' atom index: each segment's slots (one per atom, Seg), the
// plan's atom statistics, and the work order over them.
static void index_segments(kv_plan* p) {
    const int32_t L = p->c->geo.num_layers;
    const std::vector<Seg>& segs = p->segs;
    std::vector<int64_t> slots(segs.size());
    int64_t atoms = 0, writes = 0;
    for (size_t k = 0; k < segs.size(); ++k) {
        slots[k] = (int64_t)L * 2 * segs[k].C * segs[k].nh;  // every slot a real atom (Seg)
        const int64_t a = (int64_t)L * 2 * segs[k].C * segs[k].nh;         // real atoms
        atoms += a;
        writes += a * segs[k].rep1;
    }
    p->st.n_atoms = atoms;
    p->st.n_atom_writes = writes;
    build_work_order(p, slots);
    p->st.n_atom_slots = p->mixed_end;  // kernel slots: atoms + the mixed order's holes
}

// a6 sizes and the remap kernel's per-request records; packed all-pool output
// offsets of kv_remap_block_tables(gpu = -1).
static void build_remap_records(kv_plan* p, const std::vector<int32_t>& rid_off) {
    const int32_t n = p->c->n_gpus, n_reqs = (int32_t)p->reqs.size();
    p->n_res.assign(n, 0);
    p->n_res_ids.assign(n, 0);
    p->recs.resize(n_reqs);
    int64_t n_moving = 0;
    for (int32_t i = 0; i < n_reqs; ++i) {
        const ReqPlan& q = p->reqs[i];
        n_moving += q.moving;
        p->recs[i] = ReqRec{q.dst.first_gpu, q.dst.degree, q.n1, q.dst_off, rid_off[i], {0, 0, 0}};
        for (int32_t r = 0; r < q.dst.degree; ++r) {
            p->n_res[q.dst.first_gpu + r] += 1;
            p->n_res_ids[q.dst.first_gpu + r] += q.n1;
        }
    }
    p->out_off.assign((size_t)n * 3, 0);
    for (int32_t g = 0, r0 = 0, i0 = 0; g < n; ++g) {
        p->out_off[3 * g + 0] = r0 + g;  // req_ptr rows: n_res[g] + 1 each
        p->out_off[3 * g + 1] = i0;
        p->out_off[3 * g + 2] = 4 * r0;
        r0 += p->n_res[g];
        i0 += p->n_res_ids[g];
    }
    p->st.n_requests = n_reqs;
    p->st.n_moving = n_moving;
}

// Device workspace: [seg_begin | seg_of | streams | buckets | segs | tables | recs | out_off | a2a_base | items], 256-byte aligned.
static void layout_workspace(kv_plan* p) {
    auto align = [](size_t x) { return (x + 255) & ~(size_t)255; };
    p->off_seg_begin = 0;
    p->off_seg_of = align(p->off_seg_begin + p->seg_begin.size() * sizeof(int64_t));
    p->off_streams = align(p->off_seg_of + p->seg_of.size() * sizeof(int32_t));
    p->off_buckets = align(p->off_streams + p->streams.size() * sizeof(MixStream));
    p->off_segs = align(p->off_buckets + p->buckets.size() * sizeof(MixBucket));
    p->off_tables = align(p->off_segs + p->segs.size() * sizeof(Seg));
    p->off_recs = align(p->off_tables + p->tables.size() * sizeof(int32_t));
    p->off_outs = align(p->off_recs + p->recs.size() * sizeof(ReqRec));
    p->off_a2a = align(p->off_outs + p->out_off.size() * sizeof(int32_t));
    p->off_items = align(p->off_a2a + p->a2a_base.size() * sizeof(int64_t));
    p->dbytes = align(p->off_items + p->items.size() * sizeof(A2AItem));
}

extern "C" kv_status kv_cache_set_multicast(kv_cache* c, kv_group team, void* const* layer_base, int32_t mode) {
    if (!c || (mode != 1 && mode != 2)) return fail(KV_ERR_INVALID_ARG, "bad kv_cache_set_multicast arguments");
    const int32_t n = c->n_gpus, L = c->geo.num_layers;
    if (team.degree < 2 || team.first_gpu < 0 || team.first_gpu % team.degree || team.first_gpu + team.degree > n)
        return fail(KV_ERR_INVALID_ARG, "team [%d, +%d) is not an aligned group of >= 2 pools", team.first_gpu,
                    team.degree);
    if (c->mc_mode && c->mc_mode != mode)
        return fail(KV_ERR_INVALID_ARG, "teams of one cache share one mode (%d registered)", c->mc_mode);
    if (c->mc_team.empty()) {
        c->mc_team.assign(n, 0);
        c->mc_base.assign((size_t)n * L, nullptr);
    }
    for (int32_t l = 0; l < L; ++l) {
        if (layer_base && !layer_base[l]) return fail(KV_ERR_INVALID_ARG, "layer %d multicast base is NULL", l);
        c->mc_base[(size_t)team.first_gpu * L + l] = layer_base ? layer_base[l] : nullptr;
    }
    c->mc_team[team.first_gpu] = layer_base ? team.degree : 0;
    bool any = false;
    for (int32_t x : c->mc_team) any = any || x;
    c->mc_mode = any ? mode : 0;
    c->mc_dirty = true;
    return KV_OK;
}

// Device copies of the multicast team tables (kv_cache_set_multicast).
static kv_status ensure_mc(kv_cache* c) {
    if (!c->mc_dirty || c->mc_team.empty()) return KV_OK;
    const int32_t n = c->n_gpus, L = c->geo.num_layers;
    if (!c->d_mc_base) CUDA_TRY(cudaMalloc(&c->d_mc_base, (size_t)n * L * sizeof(void*)));
    if (!c->d_mc_team) CUDA_TRY(cudaMalloc(&c->d_mc_team, (size_t)n * sizeof(int32_t)));
    CUDA_TRY(cudaMemcpy(c->d_mc_base, c->mc_base.data(), (size_t)n * L * sizeof(void*), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMemcpy(c->d_mc_team, c->mc_team.data(), (size_t)n * sizeof(int32_t), cudaMemcpyHostToDevice));
    c->mc_dirty = false;
    return KV_OK;
}

extern "C" kv_status kv_cache_set_strict(kv_cache* c, int32_t strict) {
    if (!c || (strict != 0 && strict != 1)) return fail(KV_ERR_INVALID_ARG, "bad kv_cache_set_strict arguments");
    c->strict = strict;
    return KV_OK;
}

extern "C" kv_status kv_cache_set_work_order(kv_cache* c, int32_t order) {
    if (!c || (order != 0 && order != 1)) return fail(KV_ERR_INVALID_ARG, "bad kv_cache_set_work_order arguments");
    c->work_order = order;
    return KV_OK;
}

extern "C" kv_status kv_plan_switch(kv_cache* c, const kv_request* reqs, int32_t n_reqs, kv_plan** out) {
    if (!c || !out || n_reqs < 0 || (n_reqs > 0 && !reqs))
        return fail(KV_ERR_INVALID_ARG, "bad kv_plan_switch arguments");
    *out = nullptr;
    int64_t total_src = 0, total_dst_bound = 0;
    kv_status vs = validate_requests(c, reqs, n_reqs, &total_src, &total_dst_bound);  // a2, no state change
    if (vs) return vs;
    kv_plan* p = new (std::nothrow) kv_plan();
    if (!p) return fail(KV_ERR_INVALID_ARG, "out of host memory");
    p->c = c;
    p->reqs.resize(n_reqs);
    p->tables.reserve((size_t)(total_src + total_dst_bound + n_reqs));
    init_requests(p, reqs, n_reqs);
    const int32_t full = allocate_destinations(p);
    if (full >= 0) {
        rollback_allocations(p, full);
        const ReqPlan& q = p->reqs[full];
        kv_status st = fail(KV_ERR_OUT_OF_BLOCKS, "request %d needs %d blocks on group [%d,+%d)", full, q.n1,
                            q.dst.first_gpu, q.dst.degree);
        delete p;
        return st;
    }
    std::vector<int32_t> rid_off, inv_off;
    rank_id_tables(p, rid_off, inv_off);
    std::vector<Seg> segs;
    std::vector<int32_t> seg_req;
    const int32_t big = build_segments(p, inv_off, segs, seg_req);
    if (big >= 0) {
        rollback_allocations(p, n_reqs);
        const int64_t atoms = (int64_t)c->geo.num_layers * 2 * ceil_div(p->reqs[big].T, c->geo.block_base) *
                              c->geo.num_kv_heads;
        kv_status st = fail(KV_ERR_INVALID_ARG, "request %d: %lld atoms exceed the 2^31 per-request limit", big,
                            (long long)atoms);
        delete p;
        return st;
    }
    build_a2a_layout(p, segs, seg_req);
    p->segs.swap(segs);
    index_segments(p);
    // the kernels index piece space with 32-bit slots and each GPU's mixed space with 31-bit ones
    bool too_big = p->seg_begin.back() >= ((int64_t)1 << 32);
    for (int32_t g = 0; g < c->n_gpus; ++g) {
        const int64_t end = g + 1 < c->n_gpus ? p->streams[g + 1].begin : p->mixed_end;
        too_big = too_big || end - p->streams[g].begin >= ((int64_t)1 << 31);
    }
    if (too_big) {
        rollback_allocations(p, n_reqs);
        kv_status st = fail(KV_ERR_INVALID_ARG, "plan of %lld atom slots exceeds the kernels' 32-bit index",
                            (long long)p->seg_begin.back());
        delete p;
        return st;
    }
    build_remap_records(p, rid_off);
    layout_workspace(p);
    c->live.insert(p);
    p->st.atom_bytes = c->atom_bytes;
    p->st.payload_bytes = p->st.n_atom_writes * c->atom_bytes;
    p->st.h2d_bytes = (int64_t)p->dbytes;
    p->st.n_segments = (int64_t)p->segs.size();
    *out = p;
    return KV_OK;
}

// Upload the cache's pool pointer table (once per device) and the plan's
// descriptors (once per plan) -- the only host->device crossing of a switch.
static kv_status ensure_device(kv_plan* p, cudaStream_t stream) {
    kv_cache* c = p->c;
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    if (c->dev >= 0 && c->dev != dev)  // plans' workspaces live in this device's pool
        return fail(KV_ERR_BAD_STATE, "cache is bound to device %d, current device is %d", c->dev, dev);
    if (c->dev < 0) {
        const size_t nbytes = c->layer_base.size() * sizeof(void*);
        CUDA_TRY(cudaMalloc(&c->d_layer_base, nbytes));
        CUDA_TRY(cudaMemcpy(c->d_layer_base, c->layer_base.data(), nbytes, cudaMemcpyHostToDevice));
        cudaMemPoolProps props{};
        props.allocType = cudaMemAllocationTypePinned;
        props.location.type = cudaMemLocationTypeDevice;
        props.location.id = dev;
        CUDA_TRY(cudaMemPoolCreate(&c->pool, &props));
        uint64_t keep = UINT64_MAX;
        CUDA_TRY(cudaMemPoolSetAttribute(c->pool, cudaMemPoolAttrReleaseThreshold, &keep));
        // pinned host buffers up front (cudaMallocHost can take tens of ms:
        // never inside a switch): the staging ring and kv_switch's landing buffer
        for (int k = 0; k < kv_cache::kStageRing; ++k) {
            CUDA_TRY(cudaMallocHost(&c->stage[k], (size_t)1 << 20));
            c->stage_bytes[k] = (size_t)1 << 20;
        }
        CUDA_TRY(cudaMallocHost(&c->back, (size_t)1 << 20));
        c->back_bytes = (size_t)1 << 20;
        c->dev = dev;
    }
    if (p->dbuf) {
        if (p->dev != dev) return fail(KV_ERR_BAD_STATE, "plan was uploaded to device %d, current is %d", p->dev, dev);
        return KV_OK;
    }
    // pinned staging from the cache's ring; a slot is reused once its
    // previous upload has been consumed by the copy engine (kStageRing
    // uploads may be in flight, e.g. the waves of kv_switch_multi)
    const int k = c->stage_next;
    c->stage_next = (k + 1) % kv_cache::kStageRing;
    if (!c->stage_ev[k]) CUDA_TRY(cudaEventCreateWithFlags(&c->stage_ev[k], cudaEventDisableTiming));
    if (c->stage_pending[k]) {
        CUDA_TRY(cudaEventSynchronize(c->stage_ev[k]));
        c->stage_pending[k] = false;
    }
    if (c->stage_bytes[k] < p->dbytes) {
        if (c->stage[k]) cudaFreeHost(c->stage[k]);
        c->stage[k] = nullptr;
        c->stage_bytes[k] = 0;
        size_t want = std::max(p->dbytes, (size_t)1 << 20);
        CUDA_TRY(cudaMallocHost(&c->stage[k], want));
        c->stage_bytes[k] = want;
    }
    char* h = static_cast<char*>(c->stage[k]);
    std::memcpy(h + p->off_seg_begin, p->seg_begin.data(), p->seg_begin.size() * sizeof(int64_t));
    if (!p->seg_of.empty()) std::memcpy(h + p->off_seg_of, p->seg_of.data(), p->seg_of.size() * sizeof(int32_t));
    if (!p->streams.empty()) std::memcpy(h + p->off_streams, p->streams.data(), p->streams.size() * sizeof(MixStream));
    if (!p->buckets.empty()) std::memcpy(h + p->off_buckets, p->buckets.data(), p->buckets.size() * sizeof(MixBucket));
    if (!p->segs.empty()) std::memcpy(h + p->off_segs, p->segs.data(), p->segs.size() * sizeof(Seg));
    if (!p->tables.empty()) std::memcpy(h + p->off_tables, p->tables.data(), p->tables.size() * sizeof(int32_t));
    if (!p->recs.empty()) std::memcpy(h + p->off_recs, p->recs.data(), p->recs.size() * sizeof(ReqRec));
    std::memcpy(h + p->off_outs, p->out_off.data(), p->out_off.size() * sizeof(int32_t));
    if (!p->a2a_base.empty()) std::memcpy(h + p->off_a2a, p->a2a_base.data(), p->a2a_base.size() * sizeof(int64_t));
    if (!p->items.empty()) std::memcpy(h + p->off_items, p->items.data(), p->items.size() * sizeof(A2AItem));
    CUDA_TRY(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p->dbuf), p->dbytes, c->pool, stream));
    CUDA_TRY(cudaMemcpyAsync(p->dbuf, h, p->dbytes, cudaMemcpyHostToDevice, stream));
    CUDA_TRY(cudaEventRecord(c->stage_ev[k], stream));
    c->stage_pending[k] = true;
    p->dev = dev;
    p->last_stream = stream;
    return KV_OK;
}

extern "C" kv_status kv_plan_upload(kv_plan* p, void* stream) {
    PLAN_CHECK(p);
    return ensure_device(p, static_cast<cudaStream_t>(stream));
}

// Launch arguments of the reshard kernel for the segments sourced on pools
// [lo, hi) (every pool: [0, n_gpus)).  Piece space and the mixed slot space
// are laid out source GPU after source GPU (build_work_order), so a range of
// pools is one contiguous range of both.
static ReshardArgs reshard_args(const kv_plan* p, int32_t lo, int32_t hi) {
    const kv_cache* c = p->c;
    ReshardArgs a{};
    a.seg_begin = reinterpret_cast<const int64_t*>(p->dbuf + p->off_seg_begin);
    a.seg_of = reinterpret_cast<const int32_t*>(p->dbuf + p->off_seg_of);
    a.streams = reinterpret_cast<const MixStream*>(p->dbuf + p->off_streams);
    a.buckets = reinterpret_cast<const MixBucket*>(p->dbuf + p->off_buckets);
    a.segs = reinterpret_cast<const Seg*>(p->dbuf + p->off_segs);
    a.tables = reinterpret_cast<const int32_t*>(p->dbuf + p->off_tables);
    a.layer_base = c->d_layer_base;
    const int32_t n = c->n_gpus;
    a.seg_lo = p->gpu_seg_lo[lo];
    a.seg_hi = p->gpu_seg_hi[hi - 1];
    a.st_lo = lo;
    a.st_hi = hi;
    a.atom_lo = p->streams[lo].begin;
    a.atom_hi = hi < n ? p->streams[hi].begin : p->mixed_end;
    // the first GPU with work (the stream search needs streams[st_lo].begin <= slot)
    while (a.st_lo + 1 < hi && p->streams[a.st_lo + 1].begin == a.atom_lo) ++a.st_lo;
    // The kernels may index piece space with the mixed slot directly (MIX =
    // false) only where the two coincide: every launched stream is a single
    // bucket AND starts at the same offset in both spaces.  An earlier GPU
    // with several buckets leaves holes in the mixed space, which shifts the
    // later GPUs' mixed offsets past their piece-space ones -- so a launch of
    // such a later single-bucket GPU alone (one process per GPU) must take
    // the mapping too.  (Found by tests/test_gpu_fuzz.py, seed 82.)
    for (int32_t g = a.st_lo; g < a.st_hi; ++g) {
        const MixStream& ms = p->streams[g];
        if (ms.nb > 1 || (ms.nb == 1 && ms.begin != p->buckets[ms.b0].start)) a.mixed = 1;
    }
    a.L = c->geo.num_layers;
    a.atom_bytes = (int32_t)c->atom_bytes;
    a.M = c->M;
    a.max_rep = 1;
    for (int32_t k = a.seg_lo; k < a.seg_hi; ++k) a.max_rep = std::max(a.max_rep, p->segs[p->seg_of[k]].rep1);
    return a;
}

static ReshardArgs reshard_args(const kv_plan* p, int32_t gpu) {
    return gpu < 0 ? reshard_args(p, 0, p->c->n_gpus) : reshard_args(p, gpu, gpu + 1);
}

extern "C" kv_status kv_reshard_range(kv_plan* p, int32_t gpu_lo, int32_t gpu_hi, void* stream_) {
    PLAN_CHECK(p);
    if (p->state != PLAN_PLANNED)
        return fail(KV_ERR_BAD_STATE, "plan already committed; its source blocks may be reused");
    const int32_t n = p->c->n_gpus;
    if (gpu_lo < 0 || gpu_hi > n || gpu_lo >= gpu_hi)
        return fail(KV_ERR_INVALID_ARG, "pool range [%d, %d) is not inside [0, %d)", gpu_lo, gpu_hi, n);
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    kv_status s = ensure_device(p, stream);
    if (s) return s;
    p->last_stream = stream;
    ReshardArgs a = reshard_args(p, gpu_lo, gpu_hi);
    s = ensure_mc(p->c);
    if (s) return s;
    if (p->c->mc_mode && (p->c->atom_bytes == 4096 || p->c->atom_bytes == 2048)) {  // NVLS team stores
        a.mc_base = p->c->d_mc_base;
        a.mc_team = p->c->d_mc_team;
        a.mc_mode = p->c->mc_mode;
    }
    // a share of the pools (one process per GPU): destinations may be peer
    // pools, released system-wide before the group barrier
    const bool part = gpu_lo > 0 || gpu_hi < n;
    a.fence_sys = part ? 1 : 0;
    a.peer = part ? 1 : 0;
    if (a.atom_hi <= a.atom_lo) return KV_OK;
    cudaError_t e = launch_reshard(a, p->dev, stream);
    if (e != cudaSuccess) return cuda_fail(e, "flykv_reshard_kernel launch");
    g_launches.fetch_add(1);
    return KV_OK;
}

extern "C" kv_status kv_reshard(kv_plan* p, int32_t gpu, void* stream_) {
    PLAN_CHECK(p);
    if (gpu < -1 || gpu >= p->c->n_gpus) return fail(KV_ERR_INVALID_ARG, "gpu %d out of range", gpu);
    return gpu < 0 ? kv_reshard_range(p, 0, p->c->n_gpus, stream_) : kv_reshard_range(p, gpu, gpu + 1, stream_);
}

extern "C" kv_status kv_reshard_staged(kv_plan* p, int32_t gpu, void* staging, int64_t staging_bytes, int32_t mode,
                                       void* stream_) {
    PLAN_CHECK(p);
    if (!staging || (mode != 1 && mode != 2)) return fail(KV_ERR_INVALID_ARG, "bad kv_reshard_staged arguments");
    if (p->state != PLAN_PLANNED) return fail(KV_ERR_BAD_STATE, "plan already committed");
    if (gpu < -1 || gpu >= p->c->n_gpus) return fail(KV_ERR_INVALID_ARG, "gpu %d out of range", gpu);
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    kv_status s = ensure_device(p, stream);
    if (s) return s;
    p->last_stream = stream;
    ReshardArgs a = reshard_args(p, gpu);
    a.peer = 1;  // LDG/STG path
    a.staged = mode;
    a.staging = static_cast<char*>(staging);
    if ((a.atom_hi - a.atom_lo) * p->c->atom_bytes > staging_bytes)
        return fail(KV_ERR_INVALID_ARG, "staging buffer too small: %lld bytes needed",
                    (long long)((a.atom_hi - a.atom_lo) * p->c->atom_bytes));
    if (a.atom_hi <= a.atom_lo) return KV_OK;
    cudaError_t e = launch_reshard(a, p->dev, stream);
    if (e != cudaSuccess) return cuda_fail(e, "flykv_reshard_kernel (staged) launch");
    g_launches.fetch_add(1);
    return KV_OK;
}

extern "C" kv_status kv_pack(kv_plan* p, int32_t src_gpu, void* buf, const int64_t* chunk_off, void* stream_) {
    PLAN_CHECK(p);
    if (!buf || !chunk_off) return fail(KV_ERR_INVALID_ARG, "bad kv_pack arguments");
    if (p->state != PLAN_PLANNED) return fail(KV_ERR_BAD_STATE, "plan already committed");
    const int32_t n = p->c->n_gpus;
    if (src_gpu < 0 || src_gpu >= n) return fail(KV_ERR_INVALID_ARG, "src_gpu %d out of range", src_gpu);
    if (n > 64) return fail(KV_ERR_INVALID_ARG, "kv_pack supports up to 64 GPUs");
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    kv_status s = ensure_device(p, stream);
    if (s) return s;
    p->last_stream = stream;
    ReshardArgs a = reshard_args(p, src_gpu);
    a.peer = 0;  // the send buffer is local: LDG/STG, or the TMA bulk ring under kv_set_reshard_impl(2)
    a.staged = 3;
    a.a2a_base = reinterpret_cast<const int64_t*>(p->dbuf + p->off_a2a);
    a.a2a_buf = static_cast<char*>(buf);
    for (int32_t d = 0; d < n; ++d) a.a2a_off[d] = chunk_off[d];
    if (a.atom_hi <= a.atom_lo) return KV_OK;
    cudaError_t e = launch_reshard(a, p->dev, stream);
    if (e != cudaSuccess) return cuda_fail(e, "flykv_reshard_kernel (pack) launch");
    g_launches.fetch_add(1);
    return KV_OK;
}

extern "C" kv_status kv_unpack(kv_plan* p, int32_t dst_gpu, const void* buf, const int64_t* chunk_off, void* stream_) {
    PLAN_CHECK(p);
    if (!buf || !chunk_off) return fail(KV_ERR_INVALID_ARG, "bad kv_unpack arguments");
    if (p->state != PLAN_PLANNED) return fail(KV_ERR_BAD_STATE, "plan already committed");
    const int32_t n = p->c->n_gpus;
    if (dst_gpu < 0 || dst_gpu >= n) return fail(KV_ERR_INVALID_ARG, "dst_gpu %d out of range", dst_gpu);
    if (n > 64) return fail(KV_ERR_INVALID_ARG, "kv_unpack supports up to 64 GPUs");
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    kv_status s = ensure_device(p, stream);
    if (s) return s;
    p->last_stream = stream;
    const kv_cache* c = p->c;
    UnpackArgs a{};
    a.segs = reinterpret_cast<const Seg*>(p->dbuf + p->off_segs);
    a.tables = reinterpret_cast<const int32_t*>(p->dbuf + p->off_tables);
    a.a2a_base = reinterpret_cast<const int64_t*>(p->dbuf + p->off_a2a);
    a.items = reinterpret_cast<const A2AItem*>(p->dbuf + p->off_items) + p->item_lo[dst_gpu];
    a.n_items = p->item_hi[dst_gpu] - p->item_lo[dst_gpu];
    a.n_atoms = p->recv_atoms[dst_gpu];
    a.layer_base = c->d_layer_base;
    a.L = c->geo.num_layers;
    a.atom_bytes = (int32_t)c->atom_bytes;
    a.M = c->M;
    a.buf = static_cast<const char*>(buf);
    for (int32_t g = 0; g < n; ++g) a.off[g] = chunk_off[g];
    if (a.n_atoms <= 0) return KV_OK;
    cudaError_t e = launch_unpack(a, p->dev, stream);
    if (e != cudaSuccess) return cuda_fail(e, "flykv_unpack_kernel launch");
    g_launches.fetch_add(1);
    return KV_OK;
}

extern "C" kv_status kv_plan_resident(const kv_plan* p, int32_t gpu, int32_t* n_resident, int32_t* n_ids) {
    PLAN_CHECK(p);
    if (gpu < -1 || gpu >= p->c->n_gpus) return fail(KV_ERR_INVALID_ARG, "bad arguments");
    if (gpu < 0) {  // totals over every pool (packed all-GPU outputs)
        int32_t a = 0, b = 0;
        for (int32_t g = 0; g < p->c->n_gpus; ++g) {
            a += p->n_res[g];
            b += p->n_res_ids[g];
        }
        if (n_resident) *n_resident = a;
        if (n_ids) *n_ids = b;
        return KV_OK;
    }
    if (n_resident) *n_resident = p->n_res[gpu];
    if (n_ids) *n_ids = p->n_res_ids[gpu];
    return KV_OK;
}

static void commit(kv_plan* p) {
    if (p->state == PLAN_COMMITTED) return;
    kv_cache* c = p->c;
    for (const ReqPlan& q : p->reqs) {
        if (!q.moving) continue;
        for (int32_t r = 0; r < q.src.degree; ++r)
            for (int32_t k = 0; k < q.n0; ++k) bit_clr(c->held[q.src.first_gpu + r], p->tables[q.src_off + k]);
    }
    p->state = PLAN_COMMITTED;
}

extern "C" kv_status kv_plan_commit(kv_plan* p) {
    PLAN_CHECK(p);
    commit(p);
    return KV_OK;
}

extern "C" kv_status kv_plan_waves(const kv_cache* c, const kv_request* reqs, int32_t n_reqs, int64_t max_wave_bytes,
                                   int32_t* wave_start, int32_t* n_waves) {
    if (!c || !wave_start || !n_waves || n_reqs < 0 || (n_reqs > 0 && !reqs) || max_wave_bytes < 0)
        return fail(KV_ERR_INVALID_ARG, "bad kv_plan_waves arguments");
    int64_t ts = 0, td = 0;
    kv_status s = validate_requests(c, reqs, n_reqs, &ts, &td);
    if (s) return s;
    const kv_geometry& G = c->geo;
    const int32_t H = G.num_kv_heads, B = G.block_base;
    Bitmaps sim = c->held;  // simulated allocator state
    std::vector<int32_t> ids;
    int32_t w = 0, start = 0;
    int64_t wave_bytes = 0;
    auto close_wave = [&](int32_t end) {  // release the wave's sources (its remap commits it)
        for (int32_t j = start; j < end; ++j) {
            const kv_request& r = reqs[j];
            if (!request_moves(r)) continue;
            for (int32_t q = 0; q < r.src.degree; ++q)
                for (int32_t k = 0; k < r.n_src_blocks; ++k) bit_clr(sim[r.src.first_gpu + q], r.src_blocks[k]);
        }
        wave_start[w++] = start;
        start = end;
        wave_bytes = 0;
    };
    for (int32_t i = 0; i < n_reqs; ++i) {
        const kv_request& r = reqs[i];
        if (!request_moves(r)) continue;
        const Layout l1 = layout_of(H, r.dst.degree);
        const int32_t n1 = (int32_t)ceil_div(r.num_tokens, (int64_t)B * l1.k);
        const int64_t bytes = (int64_t)G.num_layers * 2 * H * ceil_div(r.num_tokens, B) * c->atom_bytes * l1.rep;
        if (max_wave_bytes > 0 && i > start && wave_bytes + bytes > max_wave_bytes) close_wave(i);
        ids.resize(n1);
        if (!alloc_lowest_in(c, sim, r.dst, n1, ids.data())) {
            if (i > start) {
                close_wave(i);
                if (alloc_lowest_in(c, sim, r.dst, n1, ids.data())) {
                    wave_bytes += bytes;
                    continue;
                }
            }
            return fail(KV_ERR_OUT_OF_BLOCKS, "request %d does not fit even in a wave of its own", i);
        }
        wave_bytes += bytes;
    }
    if (n_reqs == 0) {  // no waves; wave_start[0] = 0 is the only entry written
        wave_start[0] = 0;
        *n_waves = 0;
        return KV_OK;
    }
    if (n_reqs > start || w == 0) close_wave(n_reqs);
    wave_start[w] = n_reqs;
    *n_waves = w;
    return KV_OK;
}

// IDs free on every GPU of g in the simulated state (the most blocks one
// allocation on g can take).
static int32_t common_free(const kv_cache* c, const Bitmaps& held, kv_group g) {
    const int32_t nb = group_min_blocks(c, g);
    int32_t cnt = 0;
    for (int32_t w = 0; w < (nb + 63) >> 6; ++w) {
        uint64_t used = 0;
        for (int32_t r = 0; r < g.degree; ++r) used |= held[g.first_gpu + r][w];
        uint64_t fr = ~used;
        const int32_t top = nb - (w << 6);
        if (top < 64) fr &= (top <= 0) ? 0ull : ((1ull << top) - 1);
        cnt += __builtin_popcountll(fr);
    }
    return cnt;
}

extern "C" kv_status kv_plan_pieces(const kv_cache* c, const kv_request* reqs, int32_t n_reqs, int64_t max_wave_bytes,
                                    int32_t cap, kv_piece* pieces, int32_t* n_pieces) {
    if (!c || !n_pieces || n_reqs < 0 || (n_reqs > 0 && !reqs) || max_wave_bytes < 0 || cap < 0 ||
        (cap > 0 && !pieces))
        return fail(KV_ERR_INVALID_ARG, "bad kv_plan_pieces arguments");
    int64_t ts = 0, td = 0;
    kv_status s = validate_requests(c, reqs, n_reqs, &ts, &td);
    if (s) return s;
    const kv_geometry& G = c->geo;
    const int32_t H = G.num_kv_heads, B = G.block_base;
    Bitmaps sim = c->held;  // simulated allocator state
    std::vector<kv_piece> out;
    std::vector<int32_t> ids;
    int32_t wave = 0;
    size_t wave_first = 0;  // first piece of the open wave
    int64_t wave_bytes = 0;
    auto close_wave = [&]() {  // the wave's remap commits it: its pieces' sources are released
        for (size_t k = wave_first; k < out.size(); ++k) {
            const kv_piece& pc = out[k];
            const kv_request& r = reqs[pc.req];
            if (!request_moves(r)) continue;
            const int32_t b0 = B * layout_of(H, r.src.degree).k;
            const int32_t lo = pc.tok0 / b0, hi = (int32_t)ceil_div(pc.tok1, b0);
            for (int32_t q = 0; q < r.src.degree; ++q)
                for (int32_t k2 = lo; k2 < hi; ++k2) bit_clr(sim[r.src.first_gpu + q], r.src_blocks[k2]);
        }
        ++wave;
        wave_first = out.size();
        wave_bytes = 0;
    };
    for (int32_t i = 0; i < n_reqs; ++i) {
        const kv_request& r = reqs[i];
        if (!request_moves(r) || r.num_tokens == 0) {  // no-ops and empty requests stay whole
            out.push_back(kv_piece{wave, i, 0, r.num_tokens});
            continue;
        }
        const Layout l0 = layout_of(H, r.src.degree), l1 = layout_of(H, r.dst.degree);
        const int32_t b1 = B * l1.k;
        // piece boundaries: whole blocks of both layouts (k is a power of two)
        const int32_t unit = B * std::max(l0.k, l1.k);
        const int64_t bytes_per_chunk = (int64_t)G.num_layers * 2 * H * c->atom_bytes * l1.rep;  // per B tokens
        int32_t t = 0;
        while (t < r.num_tokens) {
            const int32_t rest = r.num_tokens - t;
            const int32_t free_ids = common_free(c, sim, r.dst);
            const int64_t room = max_wave_bytes > 0 ? max_wave_bytes - wave_bytes : INT64_MAX;
            int32_t len = 0;
            if (ceil_div(rest, b1) <= free_ids && ceil_div(rest, B) * bytes_per_chunk <= room) {
                len = rest;  // the whole remainder fits this wave
            } else if (out.size() > wave_first) {
                close_wave();  // a new wave first: the open one's sources are released at its commit
                continue;
            } else {  // even a fresh wave cannot take the remainder: the largest whole-unit prefix that fits
                int64_t units = std::min<int64_t>(rest / unit, (int64_t)free_ids / (unit / b1));
                if (max_wave_bytes > 0) units = std::min<int64_t>(units, room / ((unit / B) * bytes_per_chunk));
                len = (int32_t)(units * unit);
                if (len == 0 && max_wave_bytes > 0 && ceil_div(std::min(rest, unit), b1) <= free_ids)
                    len = std::min(rest, unit);  // one unit exceeds the byte bound on its own: take it alone
                if (len == 0)
                    return fail(KV_ERR_OUT_OF_BLOCKS, "request %d: no room for %d more tokens even in a wave of "
                                "its own", i, rest);
            }
            ids.resize(ceil_div(len, b1));
            if (!alloc_lowest_in(c, sim, r.dst, (int32_t)ids.size(), ids.data()))
                return fail(KV_ERR_OUT_OF_BLOCKS, "request %d: internal allocation mismatch", i);
            out.push_back(kv_piece{wave, i, t, t + len});
            wave_bytes += ceil_div(len, B) * bytes_per_chunk;
            t += len;
        }
    }
    *n_pieces = (int32_t)out.size();
    if ((int32_t)out.size() > cap)
        return fail(KV_ERR_INVALID_ARG, "%d pieces do not fit in cap %d (retry with *n_pieces)", (int32_t)out.size(), cap);
    std::copy(out.begin(), out.end(), pieces);
    return KV_OK;
}

extern "C" kv_status kv_suggest_rank_ids(const kv_cache* c, const kv_request* reqs, int32_t n_reqs, kv_group dst,
                                         int32_t* out) {
    if (!c || !out || n_reqs < 0 || (n_reqs > 0 && !reqs)) return fail(KV_ERR_INVALID_ARG, "bad arguments");
    kv_status s = check_group(c, dst);
    if (s) return s;
    const int32_t p = dst.degree, H = c->geo.num_kv_heads, B = c->geo.block_base, L = c->geo.num_layers;
    for (int32_t m = 0; m < p; ++m) out[m] = m;
    if (p > 16) return KV_OK;  // exact assignment only up to 16 members; identity beyond
    const Layout l1 = layout_of(H, p);
    // gain[m][r]: bytes already on member m's GPU that rank ID r would own
    std::vector<int64_t> gain((size_t)p * p, 0);
    for (int32_t i = 0; i < n_reqs; ++i) {
        const kv_request& r = reqs[i];
        if (r.dst.first_gpu != dst.first_gpu || r.dst.degree != p) continue;
        s = check_group(c, r.src);
        if (s) return s;
        const Layout l0 = layout_of(H, r.src.degree);
        const int64_t head_bytes = (int64_t)L * 2 * ceil_div(r.num_tokens, B) * c->atom_bytes;
        for (int32_t rid = 0; rid < p; ++rid) {
            const int32_t h0 = first_head_of_rank(l1, rid);
            const int32_t nh = l1.rep == 1 ? l1.hloc : 1;
            for (int32_t h = h0; h < h0 + nh; ++h) {
                const int32_t src_rid = owner_rank(l0, h, 0);  // canonical replica (R10)
                int32_t sm = src_rid;
                if (r.src_rank_ids)
                    for (int32_t q = 0; q < r.src.degree; ++q)
                        if (r.src_rank_ids[q] == src_rid) sm = q;
                const int32_t g = r.src.first_gpu + sm;
                if (g >= dst.first_gpu && g < dst.first_gpu + p) gain[(size_t)(g - dst.first_gpu) * p + rid] += head_bytes;
            }
        }
    }
    // exact assignment by DP over subsets of rank IDs (members in order)
    const uint32_t full = (1u << p) - 1;
    std::vector<int64_t> dp((size_t)full + 1, -1);
    std::vector<int8_t> parent((size_t)full + 1, -1);
    dp[0] = 0;
    for (uint32_t mask = 0; mask < full; ++mask) {
        if (dp[mask] < 0) continue;
        const int32_t m = __builtin_popcount(mask);
        for (int32_t rid = 0; rid < p; ++rid) {
            if (mask & (1u << rid)) continue;
            const uint32_t nm = mask | (1u << rid);
            const int64_t v = dp[mask] + gain[(size_t)m * p + rid];
            if (v > dp[nm]) {
                dp[nm] = v;
                parent[nm] = (int8_t)rid;
            }
        }
    }
    uint32_t mask = full;
    for (int32_t m = p - 1; m >= 0; --m) {
        const int32_t rid = parent[mask];
        out[m] = rid;
        mask ^= 1u << rid;
    }
    return KV_OK;
}

extern "C" kv_status kv_remap_block_tables(kv_plan* p, int32_t gpu, int32_t* req_ptr, int32_t* block_ids,
                                           int32_t* per_req_meta, void* stream_) {
    PLAN_CHECK(p);
    kv_cache* c = p->c;
    if (gpu < -1 || gpu >= c->n_gpus) return fail(KV_ERR_INVALID_ARG, "gpu %d out of range", gpu);
    int32_t n_res = 0, n_ids = 0;
    kv_plan_resident(p, gpu, &n_res, &n_ids);
    if (!req_ptr || (n_res > 0 && (!per_req_meta || (n_ids > 0 && !block_ids))))
        return fail(KV_ERR_INVALID_ARG, "NULL output buffer");
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    kv_status s = ensure_device(p, stream);
    if (s) return s;
    p->last_stream = stream;
    commit(p);
    RemapArgs a{};
    a.reqs = reinterpret_cast<const ReqRec*>(p->dbuf + p->off_recs);
    a.tables = reinterpret_cast<const int32_t*>(p->dbuf + p->off_tables);
    a.out_off = gpu < 0 ? reinterpret_cast<const int32_t*>(p->dbuf + p->off_outs) : nullptr;
    a.n_reqs = (int32_t)p->reqs.size();
    a.gpu = gpu;
    a.H = c->geo.num_kv_heads;
    a.B = c->geo.block_base;
    a.req_ptr = req_ptr;
    a.block_ids = block_ids;
    a.meta = per_req_meta;
    cudaError_t e = launch_remap(a, gpu < 0 ? c->n_gpus : 1, stream);
    if (e != cudaSuccess) return cuda_fail(e, "flykv_remap_kernel launch");
    g_launches.fetch_add(1);
    return KV_OK;
}

extern "C" kv_status kv_plan_packed_offsets(const kv_plan* p, int32_t* out, int64_t* totals) {
    PLAN_CHECK(p);
    if (!out) return fail(KV_ERR_INVALID_ARG, "out is NULL");
    std::memcpy(out, p->out_off.data(), p->out_off.size() * sizeof(int32_t));
    if (totals) {
        int32_t r = 0, i = 0;
        kv_plan_resident(p, -1, &r, &i);
        totals[0] = (int64_t)r + p->c->n_gpus;
        totals[1] = i;
        totals[2] = 4 * (int64_t)r;
    }
    return KV_OK;
}

extern "C" kv_status kv_plan_dst_tables(const kv_plan* p, int32_t* dst_ptr, int32_t* dst_ids) {
    if (!p || !dst_ptr) return fail(KV_ERR_INVALID_ARG, "bad arguments");
    dst_ptr[0] = 0;
    for (size_t i = 0; i < p->reqs.size(); ++i) {
        const ReqPlan& q = p->reqs[i];
        if (dst_ids)
            std::memcpy(dst_ids + dst_ptr[i], p->tables.data() + q.dst_off, (size_t)q.n1 * sizeof(int32_t));
        dst_ptr[i + 1] = dst_ptr[i] + q.n1;
    }
    return KV_OK;
}

extern "C" kv_status kv_plan_get_stats(const kv_plan* p, kv_plan_stats* st, int64_t* bytes_matrix) {
    if (!p) return fail(KV_ERR_INVALID_ARG, "plan is NULL");
    if (st) *st = p->st;
    if (bytes_matrix) std::memcpy(bytes_matrix, p->bytes.data(), p->bytes.size() * sizeof(int64_t));
    return KV_OK;
}

extern "C" kv_status kv_plan_a2a_offsets(const kv_plan* p, int64_t* send_off, int64_t* recv_off, int64_t* packed) {
    PLAN_CHECK(p);
    const int32_t n = p->c->n_gpus;
    const std::vector<int64_t>& m = p->bytes;  // m[s*n + d]
    int64_t flat = 0;
    for (int32_t s = 0; s < n; ++s) {
        int64_t acc = 0;
        for (int32_t d = 0; d < n; ++d) {
            if (send_off) send_off[(size_t)s * n + d] = acc;
            if (packed) packed[(size_t)s * n + d] = flat;
            acc += m[(size_t)s * n + d];
            flat += m[(size_t)s * n + d];
        }
    }
    if (recv_off)
        for (int32_t d = 0; d < n; ++d) {
            int64_t acc = 0;
            for (int32_t s = 0; s < n; ++s) {
                recv_off[(size_t)d * n + s] = acc;
                acc += m[(size_t)s * n + d];
            }
        }
    return KV_OK;
}

// Bytes of slots [a0, a1) of the segment at piece-space position k: destination bytes
// per GPU (replicas included) and, in column n, source reads.
static void count_piece(const kv_plan* p, int32_t k, int64_t a0, int64_t a1, int64_t* row_out) {
    const int32_t n = p->c->n_gpus;
    const int64_t ab = p->c->atom_bytes;
    const Seg& sg = p->segs[p->seg_of[k]];
    const int64_t per = (int64_t)sg.C * sg.nh;           // slots per (layer, K/V)
    const int64_t kk = sg.C - (int64_t)(sg.J1 - 1) * sg.k1; // chunks of the last destination block
    for (int64_t lkv = a0 / per; lkv * per < a1; ++lkv)
        for (int64_t jb = std::max<int64_t>(0, (a0 - lkv * per) / ((int64_t)sg.nh * sg.k1)); jb < sg.J1; ++jb) {
            const int64_t kj = jb == sg.J1 - 1 ? kk : sg.k1;
            const int64_t b0 = lkv * per + jb * sg.nh * sg.k1;     // first slot of destination block jb
            if (b0 >= a1) break;
            const int64_t o0 = std::max<int64_t>(a0 - b0, 0), o1 = std::min<int64_t>(a1 - b0, sg.nh * kj);
            if (o1 <= o0) continue;
            for (int64_t hh = o0 / kj; hh * kj < o1; ++hh) {
                const int64_t cnt = std::min<int64_t>(o1, (hh + 1) * kj) - std::max<int64_t>(o0, hh * kj);
                const int32_t h = sg.h0 + (int32_t)hh;
                row_out[n] += cnt * ab;
                for (int32_t rj = 0; rj < sg.rep1; ++rj) {
                    const int32_t rid = sg.rep1 == 1 ? h / sg.hloc1 : h * sg.rep1 + rj;
                    const int32_t m = sg.dst_inv < 0 ? rid : p->tables[sg.dst_inv + rid];
                    row_out[sg.dst_g0 + m] += cnt * ab;
                }
            }
        }
}

// Piece-space slot range [b0, b1) (global) within positions [lo, hi).
static void count_piece_range(const kv_plan* p, int32_t lo, int32_t hi, int64_t b0, int64_t b1, int64_t* row_out) {
    auto it = std::upper_bound(p->seg_begin.begin() + lo, p->seg_begin.begin() + hi, b0);
    for (int32_t k = (int32_t)(it - p->seg_begin.begin()) - 1; k < hi && p->seg_begin[k] < b1; ++k) {
        const int64_t s0 = std::max(b0, p->seg_begin[k]), s1 = std::min(b1, p->seg_begin[k + 1]);
        if (s1 > s0) count_piece(p, k, s0 - p->seg_begin[k], s1 - p->seg_begin[k], row_out);
    }
}

extern "C" kv_status kv_plan_work_order(const kv_plan* p, int32_t gpu, int32_t* n_rows, int64_t* out) {
    PLAN_CHECK(p);
    if (!n_rows || gpu < 0 || gpu >= p->c->n_gpus) return fail(KV_ERR_INVALID_ARG, "bad kv_plan_work_order arguments");
    const int32_t n = p->c->n_gpus;
    const MixStream& ms = p->streams[gpu];
    const int64_t len = (gpu + 1 < n ? p->streams[gpu + 1].begin : p->mixed_end) - ms.begin;
    const int64_t rows = ceil_div(len, kQuantumSlots);
    *n_rows = (int32_t)rows;
    if (!out) return KV_OK;
    std::memset(out, 0, sizeof(int64_t) * (size_t)rows * (n + 1));
    const int32_t lo = p->gpu_seg_lo[gpu], hi = p->gpu_seg_hi[gpu];
    for (int64_t r = 0; r < rows; ++r) {
        int64_t* row_out = out + (size_t)r * (n + 1);
        const int64_t x0 = r * kQuantumSlots, x1 = std::min(len, x0 + kQuantumSlots);
        for (int64_t q = x0 / ms.Qs; q * ms.Qs < x1; ++q)
            for (int32_t b = ms.b0; b < ms.b0 + ms.nb; ++b) {
                const MixBucket& mb = p->buckets[b];
                // mixed slots [q*Qs + P, q*Qs + P + u) hold bucket slots [q*u, q*u + u)
                const int64_t m0 = std::max(x0, q * ms.Qs + mb.P), m1 = std::min(x1, q * ms.Qs + mb.P + mb.u);
                if (m1 <= m0) continue;
                const int64_t o0 = q * mb.u + (m0 - q * ms.Qs - mb.P);
                const int64_t o1 = std::min(mb.size, o0 + (m1 - m0));
                if (o1 > o0) count_piece_range(p, lo, hi, mb.start + o0, mb.start + o1, row_out);
            }
    }
    return KV_OK;
}

extern "C" void kv_plan_destroy(kv_plan* p) {
    if (!p) return;
    if (!p->c) {  // detached by kv_cache_destroy: device memory already released
        delete p;
        return;
    }
    p->c->live.erase(p);
    if (p->h_out.capacity() && p->c->spare_h.size() < 4) {
        p->h_out.clear();
        p->c->spare_h.push_back(std::move(p->h_out));
    }
    if (p->state == PLAN_PLANNED) rollback_allocations(p, (int32_t)p->reqs.size());
    if (p->dbuf) cudaFreeAsync(p->dbuf, p->last_stream);
    if (p->d_out) cudaFreeAsync(p->d_out, p->last_stream);
    delete p;
}

// R10 strict mode: (request, head, replica >= 1) items of the plan's moving
// requests whose source degree exceeds H.
static std::vector<ReplicaItem> replica_items(const kv_plan* p) {
    std::vector<ReplicaItem> items;
    const int32_t H = p->c->geo.num_kv_heads, B = p->c->geo.block_base;
    for (const ReqPlan& q : p->reqs) {
        if (!q.moving || q.src.degree <= H || q.T <= 0) continue;
        const Layout l0 = layout_of(H, q.src.degree);
        int32_t member_of[64];
        for (int32_t m = 0; m < q.src.degree; ++m) member_of[q.src_rid[m]] = m;
        for (int32_t h = 0; h < H; ++h)
            for (int32_t j = 1; j < l0.rep; ++j)
                items.push_back(ReplicaItem{q.src.first_gpu + member_of[h * l0.rep],
                                            q.src.first_gpu + member_of[h * l0.rep + j], q.src_off, l0.k,
                                            (int32_t)ceil_div(q.T, B), q.T});
    }
    return items;
}

extern "C" kv_status kv_verify_replicas(kv_plan* p, void* stream_, int64_t* mismatches, uint64_t* first) {
    PLAN_CHECK(p);
    if (!mismatches) return fail(KV_ERR_INVALID_ARG, "mismatches is NULL");
    if (p->state != PLAN_PLANNED) return fail(KV_ERR_BAD_STATE, "plan already committed; its sources may be reused");
    *mismatches = 0;
    if (first) *first = UINT64_MAX;
    const std::vector<ReplicaItem> items = replica_items(p);
    if (items.empty()) return KV_OK;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    kv_status s = ensure_device(p, stream);
    if (s) return s;
    kv_cache* c = p->c;
    const size_t ib = items.size() * sizeof(ReplicaItem), ob = 256;
    char* d = nullptr;
    CUDA_TRY(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&d), ib + ob, c->pool, stream));
    unsigned long long init[2] = {0ull, ~0ull}, out[2] = {0ull, ~0ull};
    cudaError_t e = cudaMemcpyAsync(d, items.data(), ib, cudaMemcpyHostToDevice, stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(d + ib, init, sizeof init, cudaMemcpyHostToDevice, stream);
    VerifyArgs a{};
    a.items = reinterpret_cast<const ReplicaItem*>(d);
    a.tables = reinterpret_cast<const int32_t*>(p->dbuf + p->off_tables);
    a.layer_base = c->d_layer_base;
    a.n_items = (int32_t)items.size();
    a.L = c->geo.num_layers;
    a.B = c->geo.block_base;
    a.atom_bytes = (int32_t)c->atom_bytes;
    a.tok_bytes = c->geo.head_dim * c->geo.elem_bytes;
    a.M = c->M;
    a.out = reinterpret_cast<unsigned long long*>(d + ib);
    if (e == cudaSuccess) e = launch_verify(a, stream);
    if (e == cudaSuccess) g_launches.fetch_add(1);
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, d + ib, sizeof out, cudaMemcpyDeviceToHost, stream);
    cudaFreeAsync(d, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(e, "kv_verify_replicas");
    *mismatches = (int64_t)out[0];
    if (first) *first = out[1];
    return KV_OK;
}

// kv_switch without its read-back: plan, upload, reshard, all-pool remap into
// plan-owned device tables (the remap commits the plan on the host).  *out
// is set when the plan exists past planning (the caller destroys it).
static inline int64_t now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch())
        .count();
}

// R10 strict mode (kv_cache_set_strict): replicated sources must agree
// before any byte moves.  Every process of a one-process-per-GPU job checks
// every item of the plan (peers' pools through their mappings), so all of
// them reach the same decision.
static kv_status strict_check(kv_plan* p, cudaStream_t stream) {
    kv_cache* c = p->c;
    if (!c->strict) return KV_OK;
    int64_t bad = 0;
    uint64_t first = 0;
    kv_status s = kv_verify_replicas(p, stream, &bad, &first);
    if (s) return s;
    if (bad)
        return fail(KV_ERR_REPLICA_MISMATCH,
                    "%lld source atoms differ from their canonical replica (first: item %llu, "
                    "layer %llu, K/V %llu, chunk %llu); nothing moved",
                    (long long)bad, (unsigned long long)((first >> 32) / (2ull * c->geo.num_layers)),
                    (unsigned long long)(((first >> 32) % (2ull * c->geo.num_layers)) >> 1),
                    (unsigned long long)((first >> 32) & 1ull), (unsigned long long)(first & 0xffffffffull));
    return KV_OK;
}

static kv_status switch_enqueue(kv_cache* c, const kv_request* reqs, int32_t n_reqs, cudaStream_t stream,
                                kv_plan** out) {
    *out = nullptr;
    kv_plan* p = nullptr;
    const int64_t t0 = now_ns();
    kv_status s = kv_plan_switch(c, reqs, n_reqs, &p);
    if (s) return s;
    const int64_t t1 = now_ns();
    p->st.t_plan_ns = t1 - t0;
    int32_t tot_res = 0, tot_ids = 0;
    kv_plan_resident(p, -1, &tot_res, &tot_ids);
    const int32_t n = c->n_gpus;
    p->out_rp = tot_res + n;
    p->out_ids = p->out_rp + tot_ids;
    const int64_t elems = p->out_ids + 4 * (int64_t)tot_res;
    auto abort_plan = [&](kv_status st) {
        kv_plan_destroy(p);
        return st;
    };
    s = ensure_device(p, stream);
    if (s) return abort_plan(s);
    p->last_stream = stream;
    s = strict_check(p, stream);
    if (s) return abort_plan(s);
    cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p->d_out), (size_t)elems * 4, c->pool, stream);
    if (e != cudaSuccess) return abort_plan(cuda_fail(e, "cudaMallocFromPoolAsync (tables)"));
    s = kv_reshard(p, -1, stream);
    if (s) return abort_plan(s);
    // a5 is stream order here: every pool is addressable from this device
    s = kv_remap_block_tables(p, -1, p->d_out, p->d_out + p->out_rp, p->d_out + p->out_ids, stream);
    p->st.t_enqueue_ns = now_ns() - t1;
    *out = p;  // the plan committed inside the remap call only if it got that far
    return s;
}

// One device->host copy of a plan's packed tables (through the cache's
// pinned buffer), then a stream sync.
static kv_status switch_read_back(kv_plan* p, cudaStream_t stream) {
    kv_cache* c = p->c;
    const int64_t elems = p->out_ids + 4 * (int64_t)(p->out_rp - c->n_gpus);
    cudaError_t e;
    if ((size_t)elems * 4 > c->back_bytes) {
        if (c->back) cudaFreeHost(c->back);
        c->back = nullptr;
        c->back_bytes = 0;
        const size_t want = std::max((size_t)elems * 4, (size_t)1 << 20);
        e = cudaMallocHost(&c->back, want);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMallocHost (tables)");
        c->back_bytes = want;
    }
    const int64_t t0 = now_ns();
    e = cudaMemcpyAsync(c->back, p->d_out, (size_t)elems * 4, cudaMemcpyDeviceToHost, stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(e, "kv_switch table read-back");
    const int64_t t1 = now_ns();
    if (p->h_out.capacity() < (size_t)elems && !c->spare_h.empty()) {  // reuse a destroyed plan's buffer
        p->h_out.swap(c->spare_h.back());
        c->spare_h.pop_back();
    }
    p->h_out.assign(static_cast<int32_t*>(c->back), static_cast<int32_t*>(c->back) + elems);
    p->st.t_wait_ns = t1 - t0;
    p->st.t_read_ns = now_ns() - t1;
    return KV_OK;
}

extern "C" kv_status kv_switch(kv_cache* c, const kv_request* reqs, int32_t n_reqs, void* stream_, kv_plan** out) {
    if (!out) return fail(KV_ERR_INVALID_ARG, "out is NULL");
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    kv_status s = switch_enqueue(c, reqs, n_reqs, stream, out);
    if (s) return s;
    return switch_read_back(*out, stream);
}

// kv_switch_range and kv_switch_range_host: plan, upload, push of the owned
// pools, then `barrier` (a5: every member's pushes have landed), then the
// owned pools' remaps and one read-back.  `barrier(plan, stream)` returns a
// status; the plan is not committed before it (the first remap commits), so
// a failed barrier rolls the plan back.
template <typename Barrier>
static kv_status switch_range_impl(kv_cache* c, const kv_request* reqs, int32_t n_reqs, int32_t gpu_lo,
                                   int32_t gpu_hi, void* stream_, kv_plan** out, Barrier&& barrier) {
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    kv_plan* p = nullptr;
    const int64_t t0 = now_ns();
    kv_status s = kv_plan_switch(c, reqs, n_reqs, &p);
    if (s) return s;
    const int64_t t1 = now_ns();
    p->st.t_plan_ns = t1 - t0;
    int32_t tot_res = 0, tot_ids = 0;
    kv_plan_resident(p, -1, &tot_res, &tot_ids);
    p->out_rp = tot_res + c->n_gpus;
    p->out_ids = p->out_rp + tot_ids;
    const int64_t elems = p->out_ids + 4 * (int64_t)tot_res;
    auto abort_plan = [&](kv_status st) {
        kv_plan_destroy(p);
        return st;
    };
    s = ensure_device(p, stream);
    if (s) return abort_plan(s);
    p->last_stream = stream;
    s = strict_check(p, stream);
    if (s) return abort_plan(s);
    cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p->d_out), (size_t)elems * 4, c->pool, stream);
    if (e != cudaSuccess) return abort_plan(cuda_fail(e, "cudaMallocFromPoolAsync (tables)"));
    s = kv_reshard_range(p, gpu_lo, gpu_hi, stream);
    if (s) return abort_plan(s);
    s = barrier(p, stream);
    if (s) return abort_plan(s);
    for (int32_t g = gpu_lo; g < gpu_hi; ++g) {  // the owned pools' tables, at their packed offsets
        const int32_t* off = p->out_off.data() + 3 * g;
        s = kv_remap_block_tables(p, g, p->d_out + off[0], p->d_out + p->out_rp + off[1],
                                  p->d_out + p->out_ids + off[2], stream);
        if (s) break;
    }
    p->st.t_enqueue_ns = now_ns() - t1;
    *out = p;  // committed by the first remap call
    if (s) return s;
    return switch_read_back(p, stream);
}

extern "C" kv_status kv_switch_range(kv_cache* c, const kv_request* reqs, int32_t n_reqs, int32_t gpu_lo,
                                     int32_t gpu_hi, uint64_t* const* barrier_flags, int32_t n_members, int32_t self,
                                     uint64_t barrier_target, int64_t timeout_ns, int32_t* barrier_status,
                                     void* stream_, kv_plan** out) {
    if (!c || !out) return fail(KV_ERR_INVALID_ARG, "bad kv_switch_range arguments");
    *out = nullptr;
    if (gpu_lo < 0 || gpu_hi > c->n_gpus || gpu_lo >= gpu_hi)
        return fail(KV_ERR_INVALID_ARG, "pool range [%d, %d) is not inside [0, %d)", gpu_lo, gpu_hi, c->n_gpus);
    if (n_members > 1 && !barrier_flags) return fail(KV_ERR_INVALID_ARG, "barrier_flags is NULL");
    return switch_range_impl(c, reqs, n_reqs, gpu_lo, gpu_hi, stream_, out, [&](kv_plan*, cudaStream_t stream) {
        if (n_members <= 1) return KV_OK;
        return kv_group_barrier(barrier_flags, n_members, self, barrier_target, timeout_ns, barrier_status, stream);
    });
}

extern "C" kv_status kv_switch_range_host(kv_cache* c, const kv_request* reqs, int32_t n_reqs, int32_t gpu_lo,
                                          int32_t gpu_hi, kv_host_barrier_fn barrier, void* barrier_ctx,
                                          void* stream_, kv_plan** out) {
    if (!c || !out) return fail(KV_ERR_INVALID_ARG, "bad kv_switch_range_host arguments");
    *out = nullptr;
    if (gpu_lo < 0 || gpu_hi > c->n_gpus || gpu_lo >= gpu_hi)
        return fail(KV_ERR_INVALID_ARG, "pool range [%d, %d) is not inside [0, %d)", gpu_lo, gpu_hi, c->n_gpus);
    return switch_range_impl(c, reqs, n_reqs, gpu_lo, gpu_hi, stream_, out, [&](kv_plan*, cudaStream_t stream) {
        if (!barrier) return KV_OK;
        // this process's pushes (peer stores end with a system-scope fence)
        // have completed before the host barrier is entered
        cudaError_t e = cudaStreamSynchronize(stream);
        if (e != cudaSuccess) return cuda_fail(e, "cudaStreamSynchronize (before the host barrier)");
        const int32_t rc = barrier(barrier_ctx);
        if (rc != 0) return fail(KV_ERR_BARRIER, "host barrier callback returned %d", rc);
        return KV_OK;
    });
}

extern "C" kv_status kv_switch_multi(kv_cache* c, const kv_request* reqs, const int32_t* wave_ptr, int32_t n_waves,
                                     void* stream_, kv_plan** plans) {
    if (!c || !wave_ptr || !plans || n_waves < 0 || (n_waves > 0 && wave_ptr[n_waves] > 0 && !reqs))
        return fail(KV_ERR_INVALID_ARG, "bad kv_switch_multi arguments");
    for (int32_t w = 0; w < n_waves; ++w) {
        plans[w] = nullptr;
        if (wave_ptr[w + 1] < wave_ptr[w] || wave_ptr[0] != 0)
            return fail(KV_ERR_INVALID_ARG, "wave_ptr must be a non-decreasing prefix starting at 0");
    }
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    // every wave is planned after the previous one committed (host state), and
    // its kernels are stream-ordered after the previous wave's: a block the
    // previous wave read as a source may be this wave's destination
    for (int32_t w = 0; w < n_waves; ++w) {
        kv_status s = switch_enqueue(c, reqs + wave_ptr[w], wave_ptr[w + 1] - wave_ptr[w], stream, &plans[w]);
        if (s) {
            // waves 0..w-1 have committed (their sources are released): read
            // their tables back so the caller keeps the only record of where
            // those requests now live; then report the failing wave's error
            const std::string why = g_err;
            if (cudaStreamSynchronize(stream) == cudaSuccess)
                for (int32_t k = 0; k < w; ++k) switch_read_back(plans[k], stream);
            g_err = why;
            return s;
        }
    }
    for (int32_t w = 0; w < n_waves; ++w) {
        kv_status s = switch_read_back(plans[w], stream);
        if (s) return s;
    }
    return KV_OK;
}

extern "C" kv_status kv_piece_request(const kv_geometry* geom, const kv_request* req, int32_t tok0, int32_t tok1,
                                      kv_request* out) {
    kv_status s = check_geometry(geom);
    if (s) return s;
    if (!req || !out) return fail(KV_ERR_INVALID_ARG, "NULL argument");
    s = check_degree(geom->num_kv_heads, req->src.degree);
    if (s) return s;
    *out = *req;
    if (tok0 == 0 && tok1 == req->num_tokens) return KV_OK;  // the whole request (also an empty one)
    const Layout l0 = layout_of(geom->num_kv_heads, req->src.degree);
    const int32_t b0 = geom->block_base * l0.k;  // source block tokens B(p0), Eq.2
    if (tok0 < 0 || tok1 <= tok0 || tok1 > req->num_tokens || tok0 % b0)
        return fail(KV_ERR_INVALID_ARG, "piece [%d, %d) of a %d-token request (source blocks of %d tokens)", tok0, tok1,
                    req->num_tokens, b0);
    const int32_t first = tok0 / b0;
    out->src_blocks = req->src_blocks ? req->src_blocks + first : nullptr;
    out->n_src_blocks = (int32_t)ceil_div(tok1, b0) - first;
    out->num_tokens = tok1 - tok0;
    return KV_OK;
}

extern "C" kv_status kv_switch_waves(kv_cache* c, const kv_request* reqs, int32_t n_reqs, int64_t max_wave_bytes,
                                     int32_t split, void* stream, int32_t cap, kv_piece* pieces, int32_t* n_pieces,
                                     kv_plan** plans, int32_t* n_waves) {
    if (!c || !n_pieces || !n_waves || cap < 0 || (cap > 0 && (!pieces || !plans)) || n_reqs < 0 ||
        (n_reqs > 0 && !reqs))
        return fail(KV_ERR_INVALID_ARG, "bad kv_switch_waves arguments");
    *n_waves = 0;
    kv_status s;
    if (split) {
        s = kv_plan_pieces(c, reqs, n_reqs, max_wave_bytes, cap, pieces, n_pieces);
        if (s) return s;
    } else {  // request-granular waves, written as whole-request pieces
        std::vector<int32_t> ws(n_reqs + 1);
        int32_t nw = 0;
        s = kv_plan_waves(c, reqs, n_reqs, max_wave_bytes, ws.data(), &nw);
        if (s) return s;
        *n_pieces = n_reqs;
        if (n_reqs > cap) return fail(KV_ERR_INVALID_ARG, "cap %d < %d pieces", cap, n_reqs);
        for (int32_t w = 0; w < nw; ++w)
            for (int32_t i = ws[w]; i < ws[w + 1]; ++i) pieces[i] = kv_piece{w, i, 0, reqs[i].num_tokens};
    }
    // each piece as a plain request (kv_plan_pieces' contract), waves back to back
    std::vector<kv_request> sub(*n_pieces);
    std::vector<int32_t> wave_ptr(1, 0);
    for (int32_t k = 0; k < *n_pieces; ++k) {
        const kv_piece& pc = pieces[k];
        kv_request r{};
        s = kv_piece_request(&c->geo, &reqs[pc.req], pc.tok0, pc.tok1, &r);
        if (s) return s;
        sub[k] = r;
        if (k > 0 && pc.wave != pieces[k - 1].wave) wave_ptr.push_back(k);
    }
    if (*n_pieces > 0) wave_ptr.push_back(*n_pieces);
    const int32_t nw = (int32_t)wave_ptr.size() - 1;
    s = kv_switch_multi(c, sub.data(), wave_ptr.data(), nw, stream, plans);
    *n_waves = nw;
    return s;
}

extern "C" kv_status kv_switch_back(kv_cache* c, const kv_plan* prev, void* stream, kv_plan** out) {
    if (!c || !prev || !out) return fail(KV_ERR_INVALID_ARG, "bad kv_switch_back arguments");
    *out = nullptr;
    if (prev->c != c) return fail(KV_ERR_INVALID_ARG, "plan belongs to another cache");
    if (prev->state != PLAN_COMMITTED) return fail(KV_ERR_BAD_STATE, "previous plan is not committed");
    // every request of prev, from its destination (table, rank IDs) back to its source
    std::vector<kv_request> reqs(prev->reqs.size());
    for (size_t i = 0; i < prev->reqs.size(); ++i) {
        const ReqPlan& q = prev->reqs[i];
        kv_request& r = reqs[i];
        r.req_id = q.req_id;
        r.num_tokens = q.T;
        r.src = q.dst;
        r.src_blocks = prev->tables.data() + q.dst_off;
        r.n_src_blocks = q.n1;
        r.dst = q.src;
        r.src_rank_ids = q.dst_rid;
        r.dst_rank_ids = q.src_rid;
    }
    return kv_switch(c, reqs.data(), (int32_t)reqs.size(), stream, out);
}

extern "C" kv_status kv_plan_tables(const kv_plan* p, int32_t gpu, int32_t on_device, const int32_t** req_ptr,
                                    const int32_t** block_ids, const int32_t** per_req_meta) {
    PLAN_CHECK(p);
    if (gpu < 0 || gpu >= p->c->n_gpus) return fail(KV_ERR_INVALID_ARG, "bad kv_plan_tables arguments");
    if (!p->d_out) return fail(KV_ERR_BAD_STATE, "plan was not executed by kv_switch");
    if (!on_device && p->h_out.empty())
        return fail(KV_ERR_BAD_STATE, "the plan's tables were not read back (its switch did not complete)");
    const int32_t* base = on_device ? p->d_out : p->h_out.data();
    const int32_t* off = p->out_off.data() + 3 * gpu;  // packed layout of kv_remap_block_tables(gpu = -1)
    if (req_ptr) *req_ptr = base + off[0];
    if (block_ids) *block_ids = base + p->out_rp + off[1];
    if (per_req_meta) *per_req_meta = base + p->out_ids + off[2];
    return KV_OK;
}

// ------------------------------------------------------------ weight views
extern "C" kv_status weight_shard_view(const kv_weight_desc* w, int32_t rank, int32_t m, kv_view* out) {
    if (!w || !out) return fail(KV_ERR_INVALID_ARG, "NULL argument");
    if (w->rows < 1 || w->cols < 1 || w->ld < w->cols || w->elem_bytes < 1)
        return fail(KV_ERR_INVALID_ARG, "bad matrix shape");
    if (m < 1 || rank < 0 || rank >= m) return fail(KV_ERR_RANK_OUT_OF_RANGE, "rank %d of %d", rank, m);
    const char* base = static_cast<const char*>(w->ptr);
    const int64_t e = w->elem_bytes;
    std::memset(out, 0, sizeof *out);
    out->elem_bytes = w->elem_bytes;
    auto rows_seg = [&](int k, int64_t r0, int64_t nr) {
        out->seg[k].ptr = base + r0 * w->ld * e;
        out->seg[k].rows = nr;
        out->seg[k].cols = w->cols;
        out->seg[k].ld = w->ld;
        out->seg[k].row0 = r0;
        out->seg[k].col0 = 0;
    };
    switch (w->kind) {
        case KV_W_COLUMN: {  // output features = rows of [out, in]
            if (w->rows % m) return fail(KV_ERR_INDIVISIBLE_EXTENT, "%lld rows / %d", (long long)w->rows, m);
            const int64_t k = w->rows / m;
            out->n_seg = 1;
            rows_seg(0, rank * k, k);
            return KV_OK;
        }
        case KV_W_ROW: {  // input features = columns of [out, in]
            if (w->cols % m) return fail(KV_ERR_INDIVISIBLE_EXTENT, "%lld cols / %d", (long long)w->cols, m);
            const int64_t k = w->cols / m;
            out->n_seg = 1;
            out->seg[0].ptr = base + rank * k * e;
            out->seg[0].rows = w->rows;
            out->seg[0].cols = k;
            out->seg[0].ld = w->ld;
            out->seg[0].row0 = 0;
            out->seg[0].col0 = rank * k;
            return KV_OK;
        }
        case KV_W_QKV: {  // stacked [Q; K; V] rows, head-aligned (R17, GQA R2)
            const int64_t Hq = w->num_q_heads, Hk = w->num_kv_heads, d = w->head_dim;
            if (Hq < 1 || Hk < 1 || d < 1 || w->rows != (Hq + 2 * Hk) * d)
                return fail(KV_ERR_INVALID_ARG, "QKV rows != (Hq + 2*Hkv) * head_dim");
            if (Hq % m) return fail(KV_ERR_INDIVISIBLE_EXTENT, "%lld query heads / %d", (long long)Hq, m);
            int64_t h0, nh;
            if (m <= Hk) {
                if (Hk % m) return fail(KV_ERR_INDIVISIBLE_EXTENT, "%lld KV heads / %d", (long long)Hk, m);
                nh = Hk / m;
                h0 = rank * nh;
            } else {
                if (m % Hk) return fail(KV_ERR_INDIVISIBLE_EXTENT, "degree %d not a multiple of %lld KV heads", m, (long long)Hk);
                nh = 1;
                h0 = rank / (m / Hk);
            }
            const int64_t q = Hq / m;
            out->n_seg = 3;
            rows_seg(0, rank * q * d, q * d);
            rows_seg(1, (Hq + h0) * d, nh * d);
            rows_seg(2, (Hq + Hk + h0) * d, nh * d);
            return KV_OK;
        }
        default:
            return fail(KV_ERR_INVALID_ARG, "unknown weight kind %d", w->kind);
    }
}

extern "C" kv_status kv_gather_view(const kv_view* v, void* dst, void* stream) {
    if (!v || !dst || v->n_seg < 1 || v->n_seg > 3) return fail(KV_ERR_INVALID_ARG, "bad view");
    GatherSeg g[3];
    int64_t off = 0;
    for (int k = 0; k < v->n_seg; ++k) {
        g[k].ptr = static_cast<const char*>(v->seg[k].ptr);
        g[k].rows = v->seg[k].rows;
        g[k].row_bytes = v->seg[k].cols * v->elem_bytes;
        g[k].ld_bytes = v->seg[k].ld * v->elem_bytes;
        g[k].out_off = off;
        off += g[k].rows * g[k].row_bytes;
    }
    cudaError_t e = launch_gather(g, v->n_seg, static_cast<char*>(dst), static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "flykv_gather_kernel launch");
    g_launches.fetch_add(1);
    return KV_OK;
}

// ------------------------------------------------------------ consumer proof
// kv_paged_decode's workspace: one per (device, stream), grown on demand;
// calls on one stream are ordered, so they can share it.  Its arrival
// counters are zeroed once and left at zero by every call.
struct DecodeWorkspace {
    char* buf = nullptr;
    size_t units = 0;
};
static std::mutex g_dec_mu;
static std::map<std::pair<int, cudaStream_t>, DecodeWorkspace> g_dec_ws;

extern "C" kv_status kv_paged_decode(const kv_geometry* geom, const void* layer_base, int32_t n_res,
                                     const int32_t* req_ptr, const int32_t* block_ids, const int32_t* per_req_meta,
                                     const int32_t* seq_lens, int32_t q_heads_local, const void* q, float* out,
                                     float scale, int32_t max_seq_len, int32_t flags, void* stream_) {
    kv_status s = check_geometry(geom);
    if (s) return s;
    if (geom->elem_bytes != 2 || (geom->head_dim != 64 && geom->head_dim != 128 && geom->head_dim != 256))
        return fail(KV_ERR_INVALID_ARG, "kv_paged_decode needs bf16 and head_dim 64/128/256");
    if (n_res < 0 || q_heads_local < 1 || max_seq_len < 0 || (flags & ~KV_DECODE_AFTER_DECODE) ||
        (n_res > 0 && (!layer_base || !req_ptr || !per_req_meta || !seq_lens || !q || !out)))
        return fail(KV_ERR_INVALID_ARG, "bad kv_paged_decode arguments");
    if (((uintptr_t)q & 15) || ((uintptr_t)layer_base & 15))
        return fail(KV_ERR_INVALID_ARG, "q and layer_base must be 16-byte aligned");
    if (n_res == 0) return KV_OK;
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    const int d = geom->head_dim;
    const int64_t split = decode_split_tokens();
    // units per request <= q_heads_local (H_loc x head tiles) x splits
    const size_t units = (size_t)n_res * (size_t)q_heads_local *
                         (size_t)std::max<int64_t>(1, (max_seq_len + split - 1) / split);
    const size_t unit_bytes = (size_t)(16 + 8 * d) * sizeof(float);
    DecodeArgs a{};
    {
        int dev = 0;
        CUDA_TRY(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(g_dec_mu);
        DecodeWorkspace& w = g_dec_ws[{dev, stream}];
        if (w.units < units) {
            cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
            CUDA_TRY(cudaStreamIsCapturing(stream, &cap));
            if (cap != cudaStreamCaptureStatusNone)   // a graph-owned buffer must not outlive its graph
                return fail(KV_ERR_BAD_STATE,
                            "kv_paged_decode: the stream's workspace (%zu units) is too small for %zu units and the "
                            "stream is capturing; call once with the same or larger sizes before capture",
                            w.units, units);
            if (w.buf) CUDA_TRY(cudaFreeAsync(w.buf, stream));
            w.buf = nullptr;
            w.units = 0;
            const size_t want = std::max(units, w.units * 2);
            CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&w.buf),
                                     want * unit_bytes + (want + 2) * sizeof(int32_t), stream));
            CUDA_TRY(cudaMemsetAsync(w.buf + want * unit_bytes, 0, (want + 2) * sizeof(int32_t), stream));
            w.units = want;
        }
        a.ws = reinterpret_cast<float*>(w.buf);
        a.counters = reinterpret_cast<int32_t*>(w.buf + w.units * unit_bytes);
        a.n_units_cap = (int64_t)w.units;
    }
    a.layer = static_cast<const char*>(layer_base);
    a.M = 2 * (int64_t)geom->num_kv_heads * geom->block_base * geom->head_dim * geom->elem_bytes;
    a.d = d;
    a.n_res = n_res;
    a.q_local = q_heads_local;
    a.req_ptr = req_ptr;
    a.block_ids = block_ids;
    a.meta = per_req_meta;
    a.seq_lens = seq_lens;
    a.q = static_cast<const __nv_bfloat16*>(q);
    a.out = out;
    a.scale = scale;
    a.max_seq = max_seq_len;
    cudaError_t e = launch_decode(a, decode_grid(d), (flags & KV_DECODE_AFTER_DECODE) != 0, stream);
    if (e != cudaSuccess) return cuda_fail(e, "flykv_paged_decode_kernel launch");
    g_launches.fetch_add(1);
    return KV_OK;
}

extern "C" kv_status kv_paged_decode_release(void* stream_) {
    cudaStream_t stream = static_cast<cudaStream_t>(stream_);
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_dec_mu);
    auto it = g_dec_ws.find({dev, stream});
    if (it == g_dec_ws.end()) return KV_OK;
    char* buf = it->second.buf;
    g_dec_ws.erase(it);
    if (buf) CUDA_TRY(cudaFreeAsync(buf, stream));
    return KV_OK;
}

// ------------------------------------------------------------ IPC (peer pools)
typedef int (*cuMemGetAddressRange_t)(unsigned long long*, size_t*, unsigned long long);

extern "C" kv_status kv_ipc_export(const void* dptr, uint8_t handle[64], uint64_t* offset) {
    if (!dptr || !handle || !offset) return fail(KV_ERR_INVALID_ARG, "NULL argument");
    static cuMemGetAddressRange_t fn = nullptr;
    if (!fn) {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
        if (!f || q != cudaDriverEntryPointSuccess) return fail(KV_ERR_CUDA, "cuMemGetAddressRange unavailable");
        fn = reinterpret_cast<cuMemGetAddressRange_t>(f);
    }
    unsigned long long base = 0;
    size_t size = 0;
    int r = fn(&base, &size, (unsigned long long)(uintptr_t)dptr);
    if (r != 0) return fail(KV_ERR_CUDA, "cuMemGetAddressRange failed (%d)", r);
    cudaIpcMemHandle_t h;
    CUDA_TRY(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    static_assert(sizeof(h) == 64, "IPC handle is 64 bytes");
    std::memcpy(handle, &h, 64);
    *offset = (uint64_t)((uintptr_t)dptr - base);
    return KV_OK;
}

extern "C" kv_status kv_ipc_import(const uint8_t handle[64], uint64_t offset, void** dptr) {
    if (!handle || !dptr) return fail(KV_ERR_INVALID_ARG, "NULL argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    void* base = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dptr = static_cast<char*>(base) + offset;
    return KV_OK;
}

extern "C" kv_status kv_ipc_close(void* dptr, uint64_t offset) {
    if (!dptr) return fail(KV_ERR_INVALID_ARG, "NULL argument");
    CUDA_TRY(cudaIpcCloseMemHandle(static_cast<char*>(dptr) - offset));
    return KV_OK;
}

extern "C" kv_status kv_stream_sync(void* stream) {
    CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    return KV_OK;
}

extern "C" kv_status kv_group_barrier(uint64_t* const* flags, int32_t n_members, int32_t self, uint64_t target,
                                      int64_t timeout_ns, int32_t* status, void* stream) {
    if (!flags || n_members < 1 || n_members > 64 || self < 0 || self >= n_members || timeout_ns <= 0)
        return fail(KV_ERR_INVALID_ARG, "bad kv_group_barrier arguments (n_members %d, self %d)", n_members, self);
    BarrierArgs a{};
    for (int32_t m = 0; m < n_members; ++m) {
        if (!flags[m]) return fail(KV_ERR_INVALID_ARG, "counter of member %d is NULL", m);
        if ((uintptr_t)flags[m] & 7) return fail(KV_ERR_INVALID_ARG, "counter of member %d is not 8-byte aligned", m);
        a.flags[m] = reinterpret_cast<unsigned long long*>(flags[m]);
    }
    a.n = n_members;
    a.self = self;
    a.target = target;
    a.timeout_ns = timeout_ns;
    a.status = status;
    cudaError_t e = launch_barrier(a, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "flykv_barrier_kernel launch");
    g_launches.fetch_add(1);
    return KV_OK;
}

extern "C" kv_status kv_group_barrier_selftest(int32_t n_members, int32_t rounds, int32_t absent, int64_t timeout_ns,
                                               int32_t* errors, int32_t* timeouts) {
    if (n_members < 1 || n_members > 64 || rounds < 1 || absent >= n_members || timeout_ns <= 0 || !errors ||
        !timeouts)
        return fail(KV_ERR_INVALID_ARG, "bad kv_group_barrier_selftest arguments (n_members %d, rounds %d)",
                    n_members, rounds);
    // counters, payload (one 128-byte line per member each), errors, timeouts
    const size_t line = 16 * sizeof(unsigned long long), bytes = 2 * (size_t)n_members * line + 2 * sizeof(int32_t);
    char* buf = nullptr;
    cudaError_t e = cudaMalloc(&buf, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc (barrier self-test)");
    cudaStream_t st = nullptr;
    kv_status s = KV_OK;
    int32_t out[2] = {0, 0};
    e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaMemsetAsync(buf, 0, bytes, st);
    if (e == cudaSuccess) {
        BarrierArgs a{};
        auto* ctr = reinterpret_cast<unsigned long long*>(buf);
        for (int32_t m = 0; m < n_members; ++m) a.flags[m] = ctr + 16 * m;
        a.n = n_members;
        a.self = 0;
        a.target = 0;
        a.timeout_ns = timeout_ns;
        a.status = nullptr;
        auto* payload = ctr + 16 * n_members;
        auto* cnt = reinterpret_cast<int32_t*>(buf + 2 * (size_t)n_members * line);
        e = launch_barrier_selftest(a, rounds, absent, payload, cnt, cnt + 1, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(out, cnt, sizeof(out), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e == cudaSuccess) g_launches.fetch_add(1);
    }
    if (e != cudaSuccess) s = cuda_fail(e, "barrier self-test");
    if (st) cudaStreamDestroy(st);
    cudaFree(buf);
    *errors = out[0];
    *timeouts = out[1];
    return s;
}

// ------------------------------------------------------------ misc
extern "C" const char* kv_strerror(kv_status s) {
    switch (s) {
        case KV_OK: return "ok";
        case KV_ERR_INVALID_ARG: return "invalid argument";
        case KV_ERR_INDIVISIBLE_DEGREE: return "degree incompatible with the KV head count";
        case KV_ERR_UNKNOWN_GROUP: return "unknown (unaligned or unsupported) group";
        case KV_ERR_RANK_OUT_OF_RANGE: return "rank out of range";
        case KV_ERR_INDIVISIBLE_EXTENT: return "extent not divisible by the degree";
        case KV_ERR_OUT_OF_BLOCKS: return "out of blocks";
        case KV_ERR_BAD_BLOCK_TABLE: return "bad block table";
        case KV_ERR_DUPLICATE_REQUEST: return "duplicate request";
        case KV_ERR_BAD_STATE: return "bad state";
        case KV_ERR_CUDA: return "CUDA error";
        case KV_ERR_REPLICA_MISMATCH: return "replicated source heads differ";
        case KV_ERR_BARRIER: return "host barrier failed";
    }
    return "unknown status";
}

extern "C" const char* kv_last_error(void) { return g_err.c_str(); }

extern "C" int64_t kv_launch_count(void) { return g_launches.load(); }

extern "C" kv_status kv_set_reshard_impl(int32_t impl, int32_t ctas_per_sm) {
    if (impl < 0 || impl > 3 || ctas_per_sm < 0 || ctas_per_sm > 32)
        return fail(KV_ERR_INVALID_ARG, "impl %d / ctas_per_sm %d", impl, ctas_per_sm);
    set_reshard_impl(impl, ctas_per_sm);
    return KV_OK;
}
