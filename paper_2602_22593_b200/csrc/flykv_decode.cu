// flykv_decode.cu -- consumer proof: paged decode attention
// that reads a pool through the per-request "stride and capacity" the KV Cache
// Adaptor hands to the attention kernel: the CSR block table of
// kv_remap_block_tables and, per request, B(p), H_loc(p) and the first KV head.
//
// Decode attention is HBM-bound: every K/V byte of the resident requests is
// read once per call, and the arithmetic per byte is small.  The contraction
// is GQA-shaped -- the G query heads that share one KV head against 16-token
// tiles of that head -- so it runs on the tensor cores with mma.sync
// m16n8k16 (bf16 in, fp32 accumulate): S^T = K Q^T (M = 16 tokens, N = 8
// query heads, K = head_dim) and O^T += V^T P^T (M = 16 head_dim rows, N = 8
// heads, K = 16 tokens).  tcgen05's smallest tiles (M = 64/128) would idle on
// an N = 8 problem that is bound by HBM, not by the tensor cores.
//   * Operands come straight from global memory into MMA fragments: the
//     head_dim index of the K and Q^T fragments is permuted so that each
//     thread loads whole 16-byte chunks (coalesced), V is loaded token-row
//     wise and its pairs re-packed along tokens with PRMT; P moves from the
//     S^T accumulator layout to the B-operand layout with movmatrix.trans.
//   * P enters the second MMA as bf16 hi + lo parts (two MMAs), so O keeps
//     ~16 mantissa bits of P.
//   * Flash-decoding: a unit = (request, local KV head, tile of 8 query
//     heads, split of 512 tokens); the 4 warps of a CTA take the split's
//     16-token tiles round-robin, fold their online-softmax states in shared
//     memory in warp order, and a request with several splits is finished by
//     the CTA that completes its last split (per-item arrival counter), which
//     folds the splits in split order.
//   * Determinism across layouts: every assignment above is a function of
//     token indices only (tiles, splits), never of B(p) or the block
//     table, and each query head's arithmetic does not depend on the other
//     heads in its tile.  A TP rank reading the re-laid-out cache therefore
//     produces bit for bit the output the DP replica produces for the same
//     heads -- which is what tests/test_gpu_consumer.py checks.
//   * Persistent grid (3 CTAs of 4 warps per SM, <= 168 registers): CTAs
//     draw units from an arrival counter (the next one while the current one
//     runs); units are enumerated on the device from seq_lens and the
//     per-request meta (chunked block scans), so the host needs only an upper
//     bound of the sequence lengths.  The workspace counters return to zero
//     at the end of every launch.
//   * Each warp stages its tiles through a 2-deep shared-memory ring
//     (cp.async, rows padded to 2D + 16 bytes: conflict-free fragment
//     reads), so one tile loads while the previous one computes.
//   * With KV_DECODE_AFTER_DECODE (the previous launch on the stream is a
//     decode grid), consecutive launches overlap through programmatic
//     dependent launch: the next grid scans its requests and runs its tiles
//     (a decode grid never writes the cache, q or the tables) and waits for
//     the previous one only before its workspace and out.  Without the flag
//     a launch waits for the previous kernel as usual.
//   * Measured (bench.py --decode): 0.65 of the HBM
//     roofline back to back, 0.45 with every (pool, layer) launch of 77 MB
//     serialized.  While the warps stream
//     their tiles the bytes move at ~0.8 of the peak; the rest is fixed cost
//     around that phase (per-unit geometry and block-table loads, folds,
//     uneven unit ends, the launch) that a ~12 us launch cannot amortise.
//     Launch shapes, split sizes, staging depth and programmatic dependent
//     launch are compile-time knobs (FLYKV_DEC_*) for sweeps.
#include <cuda_bf16.h>

#include "flykv_internal.h"

namespace flykv {

namespace {

constexpr int kTile = 16;                 // tokens per MMA tile
#ifndef FLYKV_DEC_SPLIT
#define FLYKV_DEC_SPLIT 512
#endif
constexpr int kSplit = FLYKV_DEC_SPLIT;   // tokens per unit
#ifndef FLYKV_DEC_WARPS
#define FLYKV_DEC_WARPS 4
#endif
#ifndef FLYKV_DEC_CTAS
#define FLYKV_DEC_CTAS 3
#endif
#ifndef FLYKV_DEC_STAGE
#define FLYKV_DEC_STAGE 2   // stages per warp (0: tiles loaded straight into registers)
#endif
#ifndef FLYKV_DEC_PDL
#define FLYKV_DEC_PDL 1     // programmatic dependent launch between consecutive decode launches
#endif
constexpr int kWarps = FLYKV_DEC_WARPS;   // warps per CTA
constexpr int kCtasPerSm = FLYKV_DEC_CTAS;  // resident CTAs per SM (launch bounds cap the registers)
constexpr int kTilesPerWarp = kSplit / 16 / kWarps;
static_assert(kTilesPerWarp >= 1 && kTilesPerWarp <= 32, "split / warps");
constexpr int kTilesPerSplit = kSplit / kTile;
constexpr int kFoldChunk = 8;             // partials folded per step by a folding CTA
constexpr int kGroup = 16;                // splits per first-level fold group

#ifdef FLYKV_DEC_TRACE
// debug: per unit, %globaltimer at phase boundaries (unit taken, geometry read, tiles done, fold done,
// end) and the SM id; read back with kv_debug_decode_trace
__device__ unsigned long long g_dec_trace[8192][8];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define DEC_TRACE(u, k)                                                       \
    do {                                                                      \
        if (threadIdx.x == 0 && (u) < 8192) g_dec_trace[(u)][(k)] = gtime(); \
    } while (0)
#else
#define DEC_TRACE(u, k) \
    do {                \
    } while (0)
#endif

__device__ __forceinline__ uint4 ldg128(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void mma_bf16(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t movtrans(uint32_t a) {
    uint32_t d;
    asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
    return d;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t d;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
    return d;
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&v);
}

__device__ __forceinline__ float bf16_lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t v) { return __uint_as_float(v & 0xffff0000u); }

// One warp's online-softmax state for its 8 head columns.
template <int D>
struct WarpState {
    float m0, m1, l0, l1;     // heads 2tig, 2tig+1 (m uniform across the 8 row groups; l partial per lane)
    float o[D / 16][4];       // O^T fragments, m-tile mi: {(d0, 2tig), (d0, 2tig+1), (d0+1, 2tig), (d0+1, 2tig+1)}
};

// One 16-token tile's operands: K rows g and g+8 (chunks tig + 4j), V rows
// 2tig, 2tig+1, 2tig+8, 2tig+9 (chunks g + 8h).
template <int D>
struct TileRegs {
    uint4 k[D / 32][2];
    uint4 v[4][D / 64];
};

// Chunk (16 bytes = 8 head_dim elements) of a K / Q row that thread tig
// holds as its j-th chunk: a bijection onto the row's D/8 chunks that keeps
// the staged shared-memory reads conflict-free (pitch = 2D + 16 bytes).
__device__ __forceinline__ int kchunk(int tig, int j) { return 2 * tig + (j & 1) + 8 * (j >> 1); }

// blk >= 0: the tile's 16 rows lie in block blk (B(p) a multiple of 16; the
// warp's block IDs were fetched up front), rows from t0 % B(p) on.  blk < 0:
// every row looks its block up (any B(p)).  Rows past T re-read row T-1
// (masked in tile_step; never stale bytes).
template <int D>
__device__ __forceinline__ void load_tile(const DecodeArgs& a, const int32_t* tab, int32_t Bp, int32_t hl, int t0,
                                          int T, int g, int tig, int32_t blk, TileRegs<D>& tr) {
    const int64_t rowb = (int64_t)D * 2;
    const int64_t half = a.M >> 1;
    const int last = T - 1 - t0;  // rows 0..last of the tile are valid
    const char* base = nullptr;
    if (blk >= 0) base = a.layer + (int64_t)blk * a.M + ((int64_t)hl * Bp + t0 % Bp) * rowb;
    auto row_ptr = [&](int x) -> const char* {
        const int xx = x <= last ? x : last;
        if (blk >= 0) return base + xx * rowb;
        const int t = t0 + xx;
        return a.layer + (int64_t)__ldg(tab + t / Bp) * a.M + ((int64_t)hl * Bp + t % Bp) * rowb;
    };
    const char* k0 = row_ptr(g);
    const char* k1 = row_ptr(g + 8);
#pragma unroll
    for (int j = 0; j < D / 32; ++j) {
        tr.k[j][0] = ldg128(k0 + kchunk(tig, j) * 16);
        tr.k[j][1] = ldg128(k1 + kchunk(tig, j) * 16);
    }
    const int tv[4] = {2 * tig, 2 * tig + 1, 2 * tig + 8, 2 * tig + 9};
#pragma unroll
    for (int x = 0; x < 4; ++x) {
        const char* vr = row_ptr(tv[x]) + half;
#pragma unroll
        for (int h = 0; h < D / 64; ++h) tr.v[x][h] = ldg128(vr + (g + 8 * h) * 16);
    }
}

__device__ __forceinline__ uint32_t word(const uint4& v, int w) {
    return w == 0 ? v.x : w == 1 ? v.y : w == 2 ? v.z : v.w;
}


// ---- shared-memory staged tiles (FLYKV_DEC_STAGE): each warp owns a ring of
// kStages stages; a stage holds the tile's 16 K rows then its 16 V rows at a
// padded pitch of 2D + 16 bytes (conflict-free fragment reads).  Lanes copy
// 16-byte chunks with cp.async (rows past T re-read row T-1), so up to
// kStages - 1 tiles are in flight while one is consumed.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 r;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(a));
    return r;
}

template <int D>
__device__ __forceinline__ void stage_tile(const DecodeArgs& a, const int32_t* tab, int32_t Bp, int32_t hl, int t0,
                                           int T, int lane, int32_t blk, uint32_t st) {
    constexpr int kRowChunks = D / 8, kPitch = 2 * D + 16;
    const int64_t rowb = (int64_t)D * 2;
    const int last = T - 1 - t0;
    const char* base = nullptr;
    if (blk >= 0) base = a.layer + (int64_t)blk * a.M + ((int64_t)hl * Bp + t0 % Bp) * rowb;
#pragma unroll
    for (int m = 0; m < 2 * 16 * kRowChunks / 32; ++m) {
        const int c = lane + 32 * m;
        const int row = c / kRowChunks, col = c % kRowChunks;   // rows 0-15 K, 16-31 V
        const int x = row & 15;
        const int xx = x <= last ? x : last;
        const char* src;
        if (blk >= 0) {
            src = base + xx * rowb;
        } else {
            const int t = t0 + xx;
            src = a.layer + (int64_t)__ldg(tab + t / Bp) * a.M + ((int64_t)hl * Bp + t % Bp) * rowb;
        }
        if (row >= 16) src += a.M >> 1;
        cp_async16(st + row * kPitch + col * 16, src + col * 16);
    }
}

template <int D>
__device__ __forceinline__ void read_tile(uint32_t st, int g, int tig, TileRegs<D>& tr) {
    constexpr int kPitch = 2 * D + 16;
#pragma unroll
    for (int j = 0; j < D / 32; ++j) {
        tr.k[j][0] = lds128(st + g * kPitch + kchunk(tig, j) * 16);
        tr.k[j][1] = lds128(st + (g + 8) * kPitch + kchunk(tig, j) * 16);
    }
    const int tv[4] = {2 * tig, 2 * tig + 1, 2 * tig + 8, 2 * tig + 9};
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int h = 0; h < D / 64; ++h) tr.v[x][h] = lds128(st + (16 + tv[x]) * kPitch + (g + 8 * h) * 16);
}

// NTL 16-token tiles with ONE online-softmax update: S^T of each tile on the
// tensor cores, the running max over all NTL*16 tokens, then O^T += V^T P^T
// per tile.  The kernel uses NTL = 1 (two tiles per update needed registers
// that cost resident CTAs: profiles/r02_decode_history.txt).
template <int D, int NTL>
__device__ __forceinline__ void tiles_step(const TileRegs<D> (&tr)[NTL], const uint32_t (&qb)[D / 16][2],
                                           const int (&t0)[NTL], int T, int g, float sl, WarpState<D>& st) {
    float sv[NTL][4];
#pragma unroll
    for (int x = 0; x < NTL; ++x) {
        // S^T = K Q^T over D/16 k-steps; k-step (j, u) uses words 2u, 2u+1 of chunk j;
        // two independent accumulator chains (u = 0 / 1), summed
        float sa[4] = {0.f, 0.f, 0.f, 0.f}, sb[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < D / 32; ++j) {
            mma_bf16(sa, word(tr[x].k[j][0], 0), word(tr[x].k[j][1], 0), word(tr[x].k[j][0], 1),
                     word(tr[x].k[j][1], 1), qb[2 * j][0], qb[2 * j][1]);
            mma_bf16(sb, word(tr[x].k[j][0], 2), word(tr[x].k[j][1], 2), word(tr[x].k[j][0], 3),
                     word(tr[x].k[j][1], 3), qb[2 * j + 1][0], qb[2 * j + 1][1]);
        }
        const bool ok0 = t0[x] + g < T, ok1 = t0[x] + g + 8 < T;
        sv[x][0] = ok0 ? (sa[0] + sb[0]) * sl : -INFINITY;   // (token g, head 2tig)
        sv[x][1] = ok0 ? (sa[1] + sb[1]) * sl : -INFINITY;   // (token g, head 2tig+1)
        sv[x][2] = ok1 ? (sa[2] + sb[2]) * sl : -INFINITY;   // (token g+8, head 2tig)
        sv[x][3] = ok1 ? (sa[3] + sb[3]) * sl : -INFINITY;   // (token g+8, head 2tig+1)
    }
    float mx0 = fmaxf(sv[0][0], sv[0][2]), mx1 = fmaxf(sv[0][1], sv[0][3]);
#pragma unroll
    for (int x = 1; x < NTL; ++x) {
        mx0 = fmaxf(mx0, fmaxf(sv[x][0], sv[x][2]));
        mx1 = fmaxf(mx1, fmaxf(sv[x][1], sv[x][3]));
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
    }
    const float mn0 = fmaxf(st.m0, mx0), mn1 = fmaxf(st.m1, mx1);
    const float c0 = exp2f(st.m0 - mn0), c1 = exp2f(st.m1 - mn1);
    st.m0 = mn0;
    st.m1 = mn1;
    float ps[NTL][4];
    float add0 = 0.f, add1 = 0.f;
#pragma unroll
    for (int x = 0; x < NTL; ++x) {
        ps[x][0] = exp2f(sv[x][0] - mn0);
        ps[x][1] = exp2f(sv[x][1] - mn1);
        ps[x][2] = exp2f(sv[x][2] - mn0);
        ps[x][3] = exp2f(sv[x][3] - mn1);
        add0 += ps[x][0] + ps[x][2];
        add1 += ps[x][1] + ps[x][3];
    }
    st.l0 = st.l0 * c0 + add0;
    st.l1 = st.l1 * c1 + add1;
    if (!__all_sync(0xffffffffu, c0 == 1.f && c1 == 1.f)) {  // x 1.0 is the identity: skipping it is exact
#pragma unroll
        for (int mi = 0; mi < D / 16; ++mi) {
            st.o[mi][0] *= c0;
            st.o[mi][1] *= c1;
            st.o[mi][2] *= c0;
            st.o[mi][3] *= c1;
        }
    }
#pragma unroll
    for (int x = 0; x < NTL; ++x) {
        // P^T as the B operand (k = tokens, n = heads): hi and lo bf16 parts,
        // tokens 0-7 and 8-15 transposed from the accumulator layout
        const uint32_t h01 = pack_bf16(ps[x][0], ps[x][1]), h23 = pack_bf16(ps[x][2], ps[x][3]);
        const uint32_t l01 = pack_bf16(ps[x][0] - bf16_lo(h01), ps[x][1] - bf16_hi(h01));
        const uint32_t l23 = pack_bf16(ps[x][2] - bf16_lo(h23), ps[x][3] - bf16_hi(h23));
        const uint32_t bh0 = movtrans(h01), bh1 = movtrans(h23), bl0 = movtrans(l01), bl1 = movtrans(l23);
        // O^T += V^T P^T: m-tile mi rows g / g+8 = words mi%4 of chunk mi/4, lo / hi halves
#pragma unroll
        for (int mi = 0; mi < D / 16; ++mi) {
            const int h = mi / 4, w = mi % 4;
            const uint32_t va = word(tr[x].v[0][h], w), vb = word(tr[x].v[1][h], w);
            const uint32_t vc = word(tr[x].v[2][h], w), vd = word(tr[x].v[3][h], w);
            const uint32_t a0 = prmt(va, vb, 0x5410), a1 = prmt(va, vb, 0x7632);
            const uint32_t a2 = prmt(vc, vd, 0x5410), a3 = prmt(vc, vd, 0x7632);
            mma_bf16(st.o[mi], a0, a1, a2, a3, bh0, bh1);
            mma_bf16(st.o[mi], a0, a1, a2, a3, bl0, bl1);
        }
    }
}

// Fold n partials (m[8], l[8], O[8][D] each) at base + k * step * kPart,
// k = 0..n-1 in order: in chunks of kFoldChunk partials every (partial, head)
// m and l are loaded in parallel and the running max is kept by sequential
// folds over shared memory (a fixed order).  Result: out[h][d] = O / L for
// the nh heads, or the folded (M, L, O) written as a partial at `to`
// (which may be base: every read happens before the write).
template <int D>
__device__ __forceinline__ void fold_partials(const float* base, int step, int n, int nh, float* out, float* to,
                                              int tid, float* sm_M, float* sm_L, float* sm_r,
                                              float (*sm_g)[8], float (*sm_pm)[8], float (*sm_pl)[8]) {
    constexpr int kPart = 16 + 8 * D;
    constexpr int kEl = 8 * D / (kWarps * 32);   // elements per thread
    const int64_t stride = (int64_t)step * kPart;
    if (tid < 8) {
        sm_M[tid] = -INFINITY;
        sm_L[tid] = 0.f;
    }
    float acc[kEl];
#pragma unroll
    for (int x = 0; x < kEl; ++x) acc[x] = 0.f;
    for (int k0 = 0; k0 < n; k0 += kFoldChunk) {
        const int kn = min(kFoldChunk, n - k0);
        __syncthreads();  // the previous chunk's readers are done
        for (int t = tid; t < 8 * kn; t += kWarps * 32) {
            const float* pk = base + (k0 + t / 8) * stride;
            sm_pm[t / 8][t % 8] = __ldcg(pk + t % 8);
            sm_pl[t / 8][t % 8] = __ldcg(pk + 8 + t % 8);
        }
        __syncthreads();
        if (tid < 8) {  // new running max; rescale factor of what was accumulated so far
            float M = sm_M[tid];
            for (int k = 0; k < kn; ++k) M = fmaxf(M, sm_pm[k][tid]);
            const float r = exp2f(sm_M[tid] - M);   // first chunk: exp2(-inf) = 0, nothing accumulated yet
            float L = sm_L[tid] * r;
            for (int k = 0; k < kn; ++k) {
                const float f = exp2f(sm_pm[k][tid] - M);
                sm_g[k][tid] = f;
                L += sm_pl[k][tid] * f;
            }
            sm_r[tid] = r;
            sm_M[tid] = M;
            sm_L[tid] = L;
        }
        __syncthreads();
#pragma unroll
        for (int x = 0; x < kEl; ++x) {
            const int e = tid + x * kWarps * 32, h = e / D;
            float o = acc[x] * sm_r[h];
            float v[kFoldChunk];
#pragma unroll
            for (int k = 0; k < kFoldChunk; ++k) v[k] = k < kn ? __ldcg(base + (k0 + k) * stride + 16 + e) : 0.f;
#pragma unroll
            for (int k = 0; k < kFoldChunk; ++k)
                if (k < kn) o += v[k] * sm_g[k][h];
            acc[x] = o;
        }
    }
    __syncthreads();   // every read of the partials is done (to may alias base)
#pragma unroll
    for (int x = 0; x < kEl; ++x) {
        const int e = tid + x * kWarps * 32, h = e / D, dd = e % D;
        if (out) {
            if (h < nh) out[(int64_t)h * D + dd] = acc[x] / sm_L[h];
        } else {
            to[16 + e] = acc[x];
        }
    }
    if (to && tid < 8) {
        to[tid] = sm_M[tid];
        to[8 + tid] = sm_L[tid];
    }
}

__device__ __forceinline__ uint32_t smem_u32addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int D>
__global__ void __launch_bounds__(kWarps * 32, D == 256 ? 2 : kCtasPerSm) flykv_paged_decode_kernel(const DecodeArgs a) {
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int g = lane >> 2, tig = lane & 3;
    extern __shared__ __align__(16) char dyn_smem[];   // FLYKV_DEC_STAGE rings
    // per-warp states for the CTA fold; chunked request scan
    // per-warp O states for the fold: inside the warp's staging ring when staged (free after its tiles)
    constexpr bool kStaged = FLYKV_DEC_STAGE > 1 && D <= 128;
    __shared__ float sm_o_static[kStaged ? 1 : kWarps][8][D];
    auto so = [&](int w) -> float(*)[D] {
        if constexpr (kStaged)
            return reinterpret_cast<float(*)[D]>(dyn_smem + w * FLYKV_DEC_STAGE * 32 * (2 * D + 16));
        else
            return sm_o_static[w];
    };
    __shared__ float sm_m[kWarps][8], sm_l[kWarps][8], sm_f[kWarps][8], sm_M[8], sm_L[8], sm_r[8];
    __shared__ float sm_g[kFoldChunk][8], sm_pm[kFoldChunk][8], sm_pl[kFoldChunk][8];
    __shared__ int sc_incl[kWarps * 32], sc_wtot[kWarps];
    __shared__ int sc_T[kWarps * 32], sc_Bp[kWarps * 32], sc_hloc[kWarps * 32], sc_rp[kWarps * 32];  // the chunk's requests
    __shared__ int sc_tot;
    __shared__ int sh_last, sh_unit;
    const float sl = a.scale * 1.4426950408889634f;  // scores in log2 units (exp2)

    int chunk_r = -kWarps * 32;  // first request of the scanned chunk
    long long chunk_u = 0;       // units before it
    int chunk_n = 0;             // units in it
    // units are taken from an arrival counter (dynamic balance; the results do not depend on which CTA
    // computes what); the last CTA to run out of units resets the counters for the next call
    // the next unit is drawn while the current one runs (its atomic latency hidden)
#if FLYKV_DEC_PDL
    // programmatic dependent launch: the next kernel on the stream may be scheduled now; it runs its
    // request scan, then waits (griddepcontrol.wait) for this grid to complete before touching
    // anything this grid reads or writes
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
    bool waited = false;
    auto pdl_wait = [&]() {   // the previous grid on the stream has completed (its workspace and out)
#if FLYKV_DEC_PDL
        if (!waited) {
            asm volatile("griddepcontrol.wait;" ::: "memory");
            waited = true;
        }
#endif
    };
    // CTA b starts with unit b; later units come from the counter, offset past the grid
    if (tid == 0) sh_unit = blockIdx.x;
    int next_u = 0;
    while (true) {
        __syncthreads();  // sh_unit is set; the previous iteration's readers are done
        const long long u = sh_unit;
        __syncthreads();  // every thread has read sh_unit
        DEC_TRACE(u, 0);
        // ---- find the unit's request: walk chunks of 128 requests forward
        bool done = false;
        while (u >= chunk_u + chunk_n) {
            chunk_u += chunk_n;
            chunk_r += kWarps * 32;
            if (chunk_r >= a.n_res) {
                done = true;
                break;
            }
            __syncthreads();  // every thread is done reading the previous chunk's scan
            const int r = chunk_r + tid;
            int x = 0;
            if (r < a.n_res) {   // the chunk's request fields, kept for the units' geometry
                const int32_t T = a.seq_lens[r], Bp = a.meta[4 * r + 1], hloc = a.meta[4 * r + 2];
                sc_T[tid] = T;
                sc_Bp[tid] = Bp;
                sc_hloc[tid] = hloc;
                sc_rp[tid] = a.req_ptr[r];
                const int32_t G = a.q_local / hloc;
                // units of request r: H_loc KV heads x ceil(G/8) head tiles x splits (one unit for T = 0,
                // which writes zeros)
                x = hloc * ((G + 7) / 8) * (T > 0 ? (T + kSplit - 1) / kSplit : 1);
            }
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            if (lane == 31) sc_wtot[wid] = x;
            __syncthreads();
            int before = 0;
            for (int w = 0; w < wid; ++w) before += sc_wtot[w];
            sc_incl[tid] = before + x;
            if (tid == kWarps * 32 - 1) sc_tot = before + x;
            __syncthreads();
            chunk_n = sc_tot;
        }
        if (done) {
            pdl_wait();
            if (tid == 0 && atomicAdd(a.counters + a.n_units_cap + 1, 1) == (int)gridDim.x - 1) {
                a.counters[a.n_units_cap] = 0;
                a.counters[a.n_units_cap + 1] = 0;
            }
            return;
        }
        // request index: first slot whose inclusive count exceeds u - chunk_u
        const int uu = (int)(u - chunk_u);
        int lo = 0, hi = kWarps * 32 - 1;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (sc_incl[mid] > uu) hi = mid;
            else lo = mid + 1;
        }
        const int r = chunk_r + lo;
        const int before = lo > 0 ? sc_incl[lo - 1] : 0;
        int local = uu - before;
        // ---- unit geometry
        const int32_t T = sc_T[lo];
        // the workspace was sized for max_seq_len: a longer request (or a unit index it pushed past the
        // workspace) is a loud error, never a stray write
        if (T > a.max_seq || u >= a.n_units_cap) __trap();
        const int32_t Bp = sc_Bp[lo];
        const int32_t hloc = sc_hloc[lo];
        const int32_t G = a.q_local / hloc;
        const int32_t NT = (G + 7) / 8;
        const int32_t S = T > 0 ? (T + kSplit - 1) / kSplit : 1;
        const int32_t s = local % S;
        local /= S;
        const int32_t nt = local % NT;
        const int32_t hl = local / NT;
        const int32_t nh = min(8, G - 8 * nt);      // heads in this tile
        const int32_t qh0 = hl * G + 8 * nt;         // first local query head of the tile
        const int32_t* tab = a.block_ids + sc_rp[lo];
        DEC_TRACE(u, 1);
        float* outp = a.out + ((int64_t)r * a.q_local + qh0) * D;
        if (T == 0) {
            pdl_wait();
            if (tid == 0) next_u = (int)gridDim.x + atomicAdd(a.counters + a.n_units_cap, 1);
            for (int i = tid; i < nh * D; i += blockDim.x) outp[i] = 0.f;
            if (tid == 0) sh_unit = next_u;
            continue;
        }
        // ---- the warp's tiles of this split: 32s + wid, +4, ...
        WarpState<D> st;
        st.m0 = st.m1 = -INFINITY;
        st.l0 = st.l1 = 0.f;
#pragma unroll
        for (int mi = 0; mi < D / 16; ++mi) st.o[mi][0] = st.o[mi][1] = st.o[mi][2] = st.o[mi][3] = 0.f;
        const int n_tiles = (T + kTile - 1) / kTile;
        const int i_end = min(n_tiles, (s + 1) * kTilesPerSplit);
        const int i0 = s * kTilesPerSplit + wid;   // the warp's tiles: i0 + kWarps * k
        // B(p) % 16 == 0: each tile lies in one block; lane k holds the block of the warp's k-th tile
        const bool fast = (Bp % kTile) == 0;
        int32_t myblk = -1;
        if (fast && lane < kTilesPerWarp) {
            const int ik = i0 + kWarps * lane;
            if (ik < i_end) myblk = __ldg(tab + (ik * kTile) / Bp);
        }
        auto blk_of = [&](int k) { return fast ? __shfl_sync(0xffffffffu, myblk, k) : -1; };
        constexpr bool kStagedLoop = FLYKV_DEC_STAGE > 1 && D <= 128;
        constexpr int kStageBytes = 32 * (2 * D + 16);
        const uint32_t ring = smem_u32addr(dyn_smem) + wid * FLYKV_DEC_STAGE * kStageBytes;
        const int nk = i0 < i_end ? (i_end - 1 - i0) / kWarps + 1 : 0;
        if constexpr (kStagedLoop) {
#pragma unroll
            for (int q = 0; q < FLYKV_DEC_STAGE - 1; ++q) {
                if (q < nk) stage_tile<D>(a, tab, Bp, hl, (i0 + kWarps * q) * kTile, T, lane, blk_of(q), ring + q * kStageBytes);
                cp_async_commit();
            }
        }
        // ---- Q^T fragments of the tile's heads (zero for padding heads)
        uint32_t qb[D / 16][2];
        {
            const bool hv = g < nh;
            const char* qrow = reinterpret_cast<const char*>(a.q + ((int64_t)r * a.q_local + qh0 + (hv ? g : 0)) * D);
#pragma unroll
            for (int j = 0; j < D / 32; ++j) {
                uint4 c = hv ? *reinterpret_cast<const uint4*>(qrow + kchunk(tig, j) * 16) : make_uint4(0, 0, 0, 0);
                qb[2 * j][0] = c.x;
                qb[2 * j][1] = c.y;
                qb[2 * j + 1][0] = c.z;
                qb[2 * j + 1][1] = c.w;
            }
        }
        if constexpr (kStagedLoop) {
            // staged ring: tiles k .. k + kStages - 2 in flight while tile k is consumed
            for (int k = 0; k < nk; ++k) {
                const int kq = k + FLYKV_DEC_STAGE - 1;
                if (kq < nk)
                    stage_tile<D>(a, tab, Bp, hl, (i0 + kWarps * kq) * kTile, T, lane, blk_of(kq),
                                  ring + (kq % FLYKV_DEC_STAGE) * kStageBytes);
                cp_async_commit();
                cp_async_wait<FLYKV_DEC_STAGE - 1>();
                __syncwarp();
                TileRegs<D> tr[1];
                read_tile<D>(ring + (k % FLYKV_DEC_STAGE) * kStageBytes, g, tig, tr[0]);
                __syncwarp();   // every lane has read the stage before it is refilled
                const int t0[1] = {(i0 + kWarps * k) * kTile};
                tiles_step<D, 1>(tr, qb, t0, T, g, sl, st);
            }
            cp_async_wait<0>();
        } else {   // head_dim 256 (or FLYKV_DEC_STAGE=0): each tile loaded into registers, then consumed
            for (int k = 0; i0 + kWarps * k < i_end; ++k) {
                const int ia = i0 + kWarps * k;
                TileRegs<D> tr[1];
                load_tile<D>(a, tab, Bp, hl, ia * kTile, T, g, tig, blk_of(k), tr[0]);
                const int t0[1] = {ia * kTile};
                tiles_step<D, 1>(tr, qb, t0, T, g, sl, st);
            }
        }
        DEC_TRACE(u, 2);
        // l: sum of the 8 row groups' partials (fixed xor order)
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
            st.l0 += __shfl_xor_sync(0xffffffffu, st.l0, o);
            st.l1 += __shfl_xor_sync(0xffffffffu, st.l1, o);
        }
        // the tiles above read only the cache, q and the tables, which the previous decode grid on the
        // stream does not write: with programmatic dependent launch they overlap that grid's tail.
        // From here on (workspace, out) the previous grid must have completed.
        pdl_wait();
        // the next unit (CTAs without a unit never touch the counter)
        if (tid == 0) {
            next_u = (int)gridDim.x + atomicAdd(a.counters + a.n_units_cap, 1);
            sh_unit = next_u;
        }
        // ---- fold the warps (warp order) in shared memory
        __syncthreads();  // the previous unit's readers are done with sm_*
#pragma unroll
        for (int mi = 0; mi < D / 16; ++mi) {
            const int d0 = 8 * (g + 8 * (mi / 4)) + 2 * (mi % 4);
            so(wid)[2 * tig][d0] = st.o[mi][0];
            so(wid)[2 * tig + 1][d0] = st.o[mi][1];
            so(wid)[2 * tig][d0 + 1] = st.o[mi][2];
            so(wid)[2 * tig + 1][d0 + 1] = st.o[mi][3];
        }
        if (g == 0) {
            sm_m[wid][2 * tig] = st.m0;
            sm_m[wid][2 * tig + 1] = st.m1;
            sm_l[wid][2 * tig] = st.l0;
            sm_l[wid][2 * tig + 1] = st.l1;
        }
        __syncthreads();
        // per head: M = max over warps, the warps' scale factors, L (warp order)
        if (tid < 8) {
            float M = -INFINITY;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sm_m[w][tid]);
            float L = 0.f;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) {
                const float f = exp2f(sm_m[w][tid] - M);  // warps without tiles: m = -inf -> 0
                sm_f[w][tid] = f;
                L += sm_l[w][tid] * f;
            }
            sm_M[tid] = M;
            sm_L[tid] = L;
        }
        __syncthreads();
        constexpr int kPart = 16 + 8 * D;
        float* part = a.ws + u * (int64_t)kPart;
        if (S > 1 && tid < 8) {
            part[tid] = sm_M[tid];
            part[8 + tid] = sm_L[tid];
        }
        for (int e = tid; e < 8 * D; e += blockDim.x) {
            const int h = e / D, dd = e % D;
            float O = 0.f;
#pragma unroll
            for (int w = 0; w < kWarps; ++w) O += so(w)[h][dd] * sm_f[w][h];
            if (S == 1) {
                if (h < nh) outp[(int64_t)h * D + dd] = O / sm_L[h];
            } else {
                part[16 + e] = O;
            }
        }
        DEC_TRACE(u, 3);
#ifdef FLYKV_DEC_TRACE
        if (tid == 0 && u < 8192) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            g_dec_trace[u][6] = smid;
            g_dec_trace[u][7] = blockIdx.x;
        }
#endif
        if (S == 1) continue;
        // ---- several splits: a fixed two-level tree.  Splits form groups of kGroup (by split index);
        // the CTA that completes a group's last split folds the group (split order); with one group
        // that is the output, otherwise the group's fold replaces its first split's partial and the
        // CTA that completes the last group folds the groups (group order).  Counters: the group's
        // first unit (groups), the item's second unit (the item).
        const long long u0 = u - s;                     // the item's first unit
        const int grp = s / kGroup, ng = (S + kGroup - 1) / kGroup;
        const int gn = min(kGroup, S - grp * kGroup);   // splits in this group
        __threadfence();
        __syncthreads();
        if (tid == 0) {
            const int old = atomicAdd(a.counters + u0 + grp * kGroup, 1);
            sh_last = old == gn - 1;
        }
        __syncthreads();
        DEC_TRACE(u, 4);
        if (!sh_last) continue;
        __threadfence();
        if (tid == 0) a.counters[u0 + grp * kGroup] = 0;   // ready for the next call on this workspace
        if (ng == 1) {
            fold_partials<D>(a.ws + u0 * (int64_t)kPart, 1, S, nh, outp, nullptr, tid, sm_M, sm_L, sm_r, sm_g, sm_pm,
                             sm_pl);
        } else {
            float* gslot = a.ws + (u0 + grp * kGroup) * (int64_t)kPart;
            fold_partials<D>(gslot, 1, gn, 8, nullptr, gslot, tid, sm_M, sm_L, sm_r, sm_g, sm_pm, sm_pl);
            __threadfence();
            __syncthreads();
            if (tid == 0) {
                const int old = atomicAdd(a.counters + u0 + 1, 1);
                sh_last = old == ng - 1;
            }
            __syncthreads();
            if (!sh_last) continue;
            __threadfence();
            if (tid == 0) a.counters[u0 + 1] = 0;
            fold_partials<D>(a.ws + u0 * (int64_t)kPart, kGroup, ng, nh, outp, nullptr, tid, sm_M, sm_L, sm_r, sm_g,
                             sm_pm, sm_pl);
        }
        DEC_TRACE(u, 5);
    }
}

}  // namespace

template <int D>
constexpr int decode_dyn_smem() {
    return (FLYKV_DEC_STAGE > 1 && D <= 128) ? kWarps * FLYKV_DEC_STAGE * 32 * (2 * D + 16) : 0;
}

template <int D>
static cudaError_t launch_decode_d(const DecodeArgs& a, int grid, bool pdl, cudaStream_t s) {
    constexpr int smem = decode_dyn_smem<D>();
    if (smem > 48 * 1024) {
        static bool done = false;   // opt in once per process
        if (!done) {
            cudaError_t e = cudaFuncSetAttribute(flykv_paged_decode_kernel<D>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            if (e != cudaSuccess) return e;
            done = true;
        }
    }
#if FLYKV_DEC_PDL
    if (pdl) {   // KV_DECODE_AFTER_DECODE: overlap with the previous launch on the stream (a decode grid)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kWarps * 32);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, flykv_paged_decode_kernel<D>, a);
    }
#else
    (void)pdl;
#endif
    flykv_paged_decode_kernel<D><<<grid, kWarps * 32, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_decode(const DecodeArgs& a, int grid, bool pdl, cudaStream_t s) {
    if (a.n_res == 0) return cudaSuccess;
    switch (a.d) {
        case 64: return launch_decode_d<64>(a, grid, pdl, s);
        case 128: return launch_decode_d<128>(a, grid, pdl, s);
        case 256: return launch_decode_d<256>(a, grid, pdl, s);
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

int decode_split_tokens() { return kSplit; }

#ifdef FLYKV_DEC_TRACE
extern "C" int kv_debug_decode_trace(unsigned long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, g_dec_trace, sizeof(unsigned long long) * 8 * (size_t)n);
}
#endif

// Persistent grid: resident CTAs per SM (2 by the launch bounds) x SMs,
// queried once per (device, head_dim).
int decode_grid(int d) {
    static int cache[64][3] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    const int k = d == 64 ? 0 : d == 128 ? 1 : 2;
    if (dev >= 0 && dev < 64 && cache[dev][k]) return cache[dev][k];
    int sms = 148, per = 2;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const void* f = d == 64    ? reinterpret_cast<const void*>(flykv_paged_decode_kernel<64>)
                    : d == 128 ? reinterpret_cast<const void*>(flykv_paged_decode_kernel<128>)
                               : reinterpret_cast<const void*>(flykv_paged_decode_kernel<256>);
    const int smem = d == 64 ? decode_dyn_smem<64>() : d == 128 ? decode_dyn_smem<128>() : decode_dyn_smem<256>();
    if (smem > 48 * 1024) cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, f, kWarps * 32, smem) != cudaSuccess || per < 1) per = 1;
    if (dev >= 0 && dev < 64) cache[dev][k] = sms * per;
    return sms * per;
}

}  // namespace flykv
