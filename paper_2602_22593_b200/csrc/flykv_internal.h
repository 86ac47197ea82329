// flykv_internal.h -- structures shared by the host planner (flykv_host.cpp)
// and the sm_100a kernels (flykv_kernels.cu).  Not part of the ABI.
#pragma once
#include <stdint.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#define FLYKV_HD __host__ __device__ __forceinline__

namespace flykv {

// Layout of one degree p for a model with H KV heads (R1-R3):
//   hloc = H_loc(p) = H/p (p <= H) or 1 (p > H)       Eq.3, R2
//   k    = B(p)/B = H/hloc  (B-token chunks per block) Eq.2
//   rep  = replicas of each head: 1 (p <= H) or p/H   R2
struct Layout {
    int32_t hloc, k, rep;
};

FLYKV_HD Layout layout_of(int32_t H, int32_t p) {
    Layout L;
    if (p <= H) { L.hloc = H / p; L.rep = 1; }
    else        { L.hloc = 1;     L.rep = p / H; }
    L.k = H / L.hloc;
    return L;
}

// Rank (within the group) of replica j of head h, and the head's index
// inside that rank's block.  Contiguous head slices (R3, Eq.1).
FLYKV_HD int32_t owner_rank(const Layout& L, int32_t h, int32_t j) {
    return L.rep == 1 ? h / L.hloc : h * L.rep + j;
}
FLYKV_HD int32_t local_head(const Layout& L, int32_t h) {
    return L.rep == 1 ? h % L.hloc : 0;
}
FLYKV_HD int32_t first_head_of_rank(const Layout& L, int32_t r) {
    return L.rep == 1 ? r * L.hloc : r / L.rep;
}

// One work segment: the atoms of one request whose canonical source replica
// (R10) is pool src_gpu.  Atom slots are in destination-major order: per
// (layer, K/V), C*nh slots, destination block j after destination block j,
// each holding its nh heads x k1 chunks (the last block, j = J1-1, its
// kk = C - (J1-1)*k1 chunks), chunk c = j*k1 + w, head h = h0 + hh:
//   a = (l*2 + kv)*C*nh + j*nh*k1 + hh*kk_j + w      (kk_j = k1, or kk for the last block)
// so consecutive slots fill one destination block sequentially (head hl's
// chunks are a contiguous B(p1)-token run, then the next head) and every
// slot is a real atom.  With k1 = 1 this is ((l*2 + kv)*C + c)*nh + hh:
// consecutive 4 KiB pieces of one source block fanning out over destination
// ranks.  (DRAM write locality is what matters: writing contiguous runs
// measured +2-3%.)
struct Seg {
    int32_t src_gpu;   // pool holding the source replica
    int32_t dst_g0;    // first pool of the destination group
    int32_t C;         // chunks = ceil(T/B)
    int32_t nh;        // heads in this segment
    int32_t h0;        // first head
    int32_t src_tab;   // offset of the source table in the plan's table array
    int32_t dst_tab;   // offset of the destination table
    int32_t hloc0, k0; // source layout
    int32_t hloc1, k1, rep1; // destination layout
    int32_t dst_inv;   // offset of the destination's member-of-rank-ID table in tables, -1 = identity
    int32_t J1;        // destination-major order: ceil(C / k1) destination blocks per (layer, K/V)
    int32_t a2a;       // offset of this segment's per-member chunk bases in the plan's a2a_base array
    int32_t pad;
};
static_assert(sizeof(Seg) == 64, "Seg is 64 bytes");

// A source GPU's mixed slot space (the kernels' atom index):
// K quanta of Qs slots; quantum q holds, for each bucket b, the bucket's
// slots [q*u_b, (q+1)*u_b) at offset P_b (slots >= size_b are holes).  So a
// sender's traffic is split over its receivers in the switch's proportions
// at every moment, not one receiver after another.
struct MixStream {
    int64_t begin;    // first mixed slot of the GPU (global)
    int32_t Qs, K;    // slots per quantum, quanta
    int32_t b0, nb;   // the GPU's buckets in the bucket array
};
struct MixBucket {
    int64_t start;    // first piece-space slot of the bucket
    int64_t size;     // its slots
    int32_t u, P;     // slots per quantum, offset inside the quantum
};

// Per-request record used by the remap kernel (a6).
struct ReqRec {
    int32_t dst_g0, dst_p, n1, dst_tab;
    int32_t dst_rid;   // offset of the destination rank IDs (rank ID of member m) in tables, -1 = identity
    int32_t pad[3];
};

struct ReshardArgs {
    // piece space: every source GPU's segments, bucket after bucket
    // (destination groups, build_work_order); piece s is segment seg_of[s]
    const int64_t* seg_begin;  // [n_seg + 1] exclusive prefix of the pieces' slot counts
    const int32_t* seg_of;     // [n_seg]
    const MixStream* streams;  // [n_gpus] mixed slot spaces
    const MixBucket* buckets;
    int32_t st_lo, st_hi;      // source GPUs of this launch
    int32_t mixed;             // 0: every launched stream is one bucket, K = 1 (mixed slot == piece-space
                               // slot, seg_of is the identity over the launched positions)
    const Seg* segs;           // [n_seg]
    const int32_t* tables;     // source + destination tables
    char* const* layer_base;   // [n_gpus * L] pool layer pointers
    int32_t seg_lo, seg_hi;    // piece range of this launch
    int64_t atom_lo, atom_hi;  // mixed slot range (streams[st_lo].begin .. end of st_hi - 1)
    int32_t L;
    int32_t atom_bytes;        // B*d*e
    int64_t M;                 // block bytes per layer
    int32_t fence_sys;         // 1: release-fence writes at system scope (peer pools)
    int32_t peer;              // 1: destinations may be peer (NVLink) mappings -> LDG/STG path
    int32_t max_rep;           // largest destination replica count in the range (launch shape)
    int32_t staged;            // comparator only: 0 fused, 1 pack into staging, 2 unpack from staging
    char* staging;             // atom (i - atom_lo) at staging + (i - atom_lo) * atom_bytes
    int32_t rep_flags;         // GQA replica stores: bit 0 = decode replicas lane-parallel, bit 1 = replica-major order
    // NVLS multicast teams (kv_cache_set_multicast): mc_team[g] = size of the
    // replica team whose first pool is g (0 = none registered), mc_base[g*L + l]
    // its layer-l multicast address; mc_mode 1 = multimem.st, 2 = emulation (st.global)
    char* const* mc_base;
    const int32_t* mc_team;
    int32_t mc_mode;
    // staged == 3 (kv_pack): every (atom, replica) goes to the send chunk of
    // its destination GPU d at a2a_buf + a2a_off[d] + (base + pos) * atom_bytes,
    // base = a2a_base[seg.a2a + member], pos = a2a_pos(...) (flykv_kernels.cu)
    const int64_t* a2a_base;
    char* a2a_buf;
    int64_t a2a_off[64];
};

// One (segment, destination member) pair received by a GPU (kv_unpack).
struct A2AItem {
    int32_t seg, m, rid, nhm;  // segment, member of its destination group, its rank ID, heads it receives
    int64_t start;             // first atom of the pair in the receiver's atom order
};

struct UnpackArgs {
    const Seg* segs;
    const int32_t* tables;
    const int64_t* a2a_base;
    const A2AItem* items;      // the receiver's pairs, ordered by source GPU then plan order
    int32_t n_items;
    int64_t n_atoms;           // atoms the receiver unpacks
    char* const* layer_base;
    int32_t L, atom_bytes;
    int64_t M;
    const char* buf;           // receive buffer
    int64_t off[64];           // byte offset in buf of the chunk from each source GPU
};

struct RemapArgs {
    const ReqRec* reqs;  // [n_reqs]
    const int32_t* tables;
    const int32_t* out_off;  // all-GPU mode: [n_gpus][3] offsets of each GPU's req_ptr / block_ids / meta; else null
    int32_t n_reqs;
    int32_t gpu;             // single-GPU mode: the pool; all-GPU mode: blockIdx.x is the pool
    int32_t H;
    int32_t B;
    int32_t* req_ptr;
    int32_t* block_ids;
    int32_t* meta;
};

struct GatherSeg {
    const char* ptr;
    int64_t rows, row_bytes, ld_bytes;
    int64_t out_off;  // byte offset of the segment in the output
};

struct DecodeArgs {
    const char* layer;          // layer region of one pool
    int64_t M;                  // block bytes per layer
    int32_t d;                  // head_dim (bf16)
    int32_t n_res, q_local;     // resident requests, local query heads
    const int32_t* req_ptr;     // CSR from kv_remap_block_tables
    const int32_t* block_ids;
    const int32_t* meta;        // {plan index, B(p), H_loc, first head}
    const int32_t* seq_lens;    // tokens per resident request
    const __nv_bfloat16* q;     // [n_res][q_local][d]
    float* out;                 // [n_res][q_local][d]
    float scale;
    int32_t max_seq;            // bound of seq_lens the workspace is sized for
    float* ws;                  // per unit: m[8], l[8], O[8][d] of one 512-token split
    int32_t* counters;          // per item (first unit index): splits done; then [n_units_cap] the
                                // next unit, [n_units_cap + 1] CTAs done; all 0 between calls
    int64_t n_units_cap;        // units the workspace holds
};

// Group completion barrier (kv_group_barrier): this process's mapping of
// every member's counter, its own index, the count to wait for.
struct BarrierArgs {
    unsigned long long* flags[64];
    int32_t n, self;
    uint64_t target;
    int64_t timeout_ns;
    int32_t* status;
};

// Strict replica check (kv_verify_replicas): one non-canonical replica of
// one head of one request, compared with the canonical (lowest-owner)
// replica over chunks c < C, valid tokens only.
struct ReplicaItem {
    int32_t gpu_c, gpu_r;   // canonical and replica pools
    int32_t src_tab, k0;    // source table offset, chunks per source block
    int32_t C, T;           // chunks, tokens
};

struct VerifyArgs {
    const ReplicaItem* items;
    const int32_t* tables;
    char* const* layer_base;
    int32_t n_items, L, B;
    int32_t atom_bytes, tok_bytes;  // B*d*e, d*e
    int64_t M;
    unsigned long long* out;        // [0] mismatching atoms, [1] smallest mismatch code
};

// Kernel launchers (flykv_kernels.cu, flykv_decode.cu).  Return cudaSuccess or the launch error.
cudaError_t launch_reshard(const ReshardArgs& a, int device, cudaStream_t s);
void set_reshard_impl(int impl, int ctas_per_sm);
cudaError_t launch_remap(const RemapArgs& a, int n_ctas, cudaStream_t s);
cudaError_t launch_gather(const GatherSeg* segs, int n_seg, char* dst, cudaStream_t s);
cudaError_t launch_decode(const DecodeArgs& a, int grid, bool pdl, cudaStream_t s);
int decode_split_tokens();
int decode_grid(int d);
cudaError_t launch_unpack(const UnpackArgs& a, int device, cudaStream_t s);
cudaError_t launch_barrier(const BarrierArgs& a, cudaStream_t s);
cudaError_t launch_barrier_selftest(const BarrierArgs& a, int32_t rounds, int32_t absent,
                                    unsigned long long* payload, int32_t* errors, int32_t* timeouts, cudaStream_t s);
cudaError_t launch_verify(const VerifyArgs& a, cudaStream_t s);

}  // namespace flykv
