// flykv_kernels.cu -- sm_100a kernels of the KV Cache Adaptor re-layout.
//
//   flykv_reshard_kernel  a4: the hot loop.  Pure data movement (no tensor
//                         cores): one warp per 4 KiB atom, 16-byte vector
//                         loads (L1 no-allocate, read-only path) of the whole
//                         atom into registers, then 16-byte stores to each
//                         destination replica -- local HBM, another virtual
//                         rank's pool on the same device, or a peer GPU's pool
//                         over NVLink 5 / NVSwitch.  Persistent grid sized to
//                         148 SMs x resident CTAs.
//   flykv_remap_kernel    a6: per-GPU CSR block table via warp-shuffle
//                         prefix sums (stream compaction of resident requests).
//   flykv_gather_kernel   a8 test utility: materialise a weight shard view.
//
// Layout terms: see include/flykv.h and flykv_internal.h.
#include "flykv_internal.h"

namespace flykv {

__device__ __forceinline__ int4 ld_stream(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ void st_stream(int4* p, const int4& v) {
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// Decoded atom: source pointer plus what is needed to form each
// destination replica's pointer (kept in scalars, no local arrays).
struct AtomAddr {
    const char* src;
    int64_t doff;      // byte offset of the atom inside a destination layer region
    int32_t l, h;      // layer, head
    int32_t dst_g0, rep1, hloc1;
};

__device__ __forceinline__ int find_seg(const int64_t* __restrict__ seg_begin, int lo, int hi,
                                        int64_t atom) {
    // invariant: seg_begin[lo] <= atom < seg_begin[hi]
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (__ldg(seg_begin + mid) <= atom) lo = mid;
        else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ void decode(const ReshardArgs& a, int64_t atom, int s, AtomAddr& out) {
    const Seg sg = a.segs[s];
    uint32_t local = (uint32_t)(atom - __ldg(a.seg_begin + s));
    uint32_t nh = (uint32_t)sg.nh, C = (uint32_t)sg.C;
    uint32_t hh = local % nh;
    local /= nh;
    uint32_t c = local % C;
    uint32_t lkv = local / C;
    uint32_t kv = lkv & 1u, l = lkv >> 1;
    int32_t h = sg.h0 + (int32_t)hh;
    const int64_t half = a.M >> 1;
    const int64_t ab = a.atom_bytes;
    // source replica (lowest owner, R10): block tab0[c / k0], chunk c % k0
    int32_t blk0 = __ldg(a.tables + sg.src_tab + (int32_t)c / sg.k0);
    int32_t w0 = (int32_t)c % sg.k0;
    out.src = a.layer_base[sg.src_gpu * a.L + l] + (int64_t)blk0 * a.M + kv * half +
              (int64_t)((h % sg.hloc0) * sg.k0 + w0) * ab;
    // destination: same formula with the destination layout and table
    int32_t blk1 = __ldg(a.tables + sg.dst_tab + (int32_t)c / sg.k1);
    int32_t w1 = (int32_t)c % sg.k1;
    out.doff = (int64_t)blk1 * a.M + kv * half + (int64_t)((h % sg.hloc1) * sg.k1 + w1) * ab;
    out.l = (int32_t)l;
    out.h = h;
    out.dst_g0 = sg.dst_g0;
    out.rep1 = sg.rep1;
    out.hloc1 = sg.hloc1;
}

// Pointer to replica j of the decoded atom (1 replica, or p/H under GQA, R2).
__device__ __forceinline__ char* dst_ptr(const ReshardArgs& a, const AtomAddr& ad, int j) {
    const int32_t r = ad.rep1 == 1 ? ad.h / ad.hloc1 : ad.h * ad.rep1 + j;
    return a.layer_base[(ad.dst_g0 + r) * a.L + ad.l] + ad.doff;
}

// VPL = 16-byte vectors per lane per atom (atom_bytes = VPL * 512); VPL = 0
// is the generic path for atoms that are a multiple of 16 but not of 512.
template <int VPL>
__global__ void __launch_bounds__(256) flykv_reshard_kernel(const ReshardArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t atom = a.atom_lo + warp; atom < a.atom_hi; atom += nwarps) {
        const int s = find_seg(a.seg_begin, a.seg_lo, a.seg_hi, atom);
        AtomAddr ad;
        decode(a, atom, s, ad);
        if constexpr (VPL > 0) {
            const int4* src = reinterpret_cast<const int4*>(ad.src) + lane;
            int4 v[VPL];
#pragma unroll
            for (int i = 0; i < VPL; ++i) v[i] = ld_stream(src + i * 32);
            for (int j = 0; j < ad.rep1; ++j) {
                int4* dst = reinterpret_cast<int4*>(dst_ptr(a, ad, j)) + lane;
#pragma unroll
                for (int i = 0; i < VPL; ++i) st_stream(dst + i * 32, v[i]);
            }
        } else {
            const int nv = a.atom_bytes >> 4;
            const int4* src = reinterpret_cast<const int4*>(ad.src);
            for (int i = lane; i < nv; i += 32) {
                int4 v = ld_stream(src + i);
                for (int j = 0; j < ad.rep1; ++j) st_stream(reinterpret_cast<int4*>(dst_ptr(a, ad, j)) + i, v);
            }
        }
    }
    if (a.fence_sys) __threadfence_system();
}

template <int VPL>
static cudaError_t launch_reshard_t(const ReshardArgs& a, int device, cudaStream_t s) {
    static int sm_count[64] = {0};
    static int per_sm[64] = {0};
    if (device < 0 || device >= 64) device = 0;
    if (sm_count[device] == 0) {
        cudaError_t e = cudaDeviceGetAttribute(&sm_count[device], cudaDevAttrMultiProcessorCount, device);
        if (e != cudaSuccess) return e;
        int nb = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, flykv_reshard_kernel<VPL>, 256, 0);
        if (e != cudaSuccess) return e;
        per_sm[device] = nb > 0 ? nb : 1;
    }
    const int64_t atoms = a.atom_hi - a.atom_lo;
    int64_t want = (atoms + 7) / 8;
    int64_t cap = (int64_t)sm_count[device] * per_sm[device];
    int grid = (int)(want < cap ? want : cap);
    if (grid < 1) grid = 1;
    flykv_reshard_kernel<VPL><<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_reshard(const ReshardArgs& a, int device, cudaStream_t s) {
    if (a.atom_hi <= a.atom_lo) return cudaSuccess;
    switch (a.atom_bytes) {
        case 512: return launch_reshard_t<1>(a, device, s);
        case 1024: return launch_reshard_t<2>(a, device, s);
        case 2048: return launch_reshard_t<4>(a, device, s);
        case 4096: return launch_reshard_t<8>(a, device, s);
        case 8192: return launch_reshard_t<16>(a, device, s);
        default: return launch_reshard_t<0>(a, device, s);
    }
}

// ----------------------------------------------------------------- remap
// One CTA of 1024 threads.  Phase 1: stream-compact the requests resident on
// `gpu` (destination group contains gpu) with two warp-shuffle inclusive
// scans (request count, block count) + a cross-warp scan in shared memory,
// carried across 1024-request tiles.  Phase 2: copy each resident request's
// destination table into its CSR row (one warp per request).
__global__ void __launch_bounds__(1024) flykv_remap_kernel(const RemapArgs a) {
    __shared__ int32_t wf[32], wc[32];
    __shared__ int32_t carry_f, carry_c;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    if (tid == 0) { carry_f = 0; carry_c = 0; }
    __syncthreads();
    for (int base = 0; base < a.n_reqs; base += 1024) {
        const int i = base + tid;
        int32_t flag = 0, cnt = 0;
        ReqRec rr = {0, 1, 0, 0};
        if (i < a.n_reqs) {
            rr = a.reqs[i];
            flag = (a.gpu >= rr.dst_g0 && a.gpu < rr.dst_g0 + rr.dst_p) ? 1 : 0;
            cnt = flag ? rr.n1 : 0;
        }
        int32_t f = flag, c = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t tf = __shfl_up_sync(0xffffffffu, f, o);
            int32_t tc = __shfl_up_sync(0xffffffffu, c, o);
            if (lane >= o) { f += tf; c += tc; }
        }
        if (lane == 31) { wf[w] = f; wc[w] = c; }
        __syncthreads();
        if (w == 0) {
            int32_t xf = wf[lane], xc = wc[lane];
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                int32_t tf = __shfl_up_sync(0xffffffffu, xf, o);
                int32_t tc = __shfl_up_sync(0xffffffffu, xc, o);
                if (lane >= o) { xf += tf; xc += tc; }
            }
            wf[lane] = xf;
            wc[lane] = xc;
        }
        __syncthreads();
        const int32_t ef = carry_f + (w ? wf[w - 1] : 0) + f - flag;
        const int32_t ec = carry_c + (w ? wc[w - 1] : 0) + c - cnt;
        if (flag) {
            Layout L = layout_of(a.H, rr.dst_p);
            a.req_ptr[ef] = ec;
            a.meta[4 * ef + 0] = i;
            a.meta[4 * ef + 1] = a.B * L.k;
            a.meta[4 * ef + 2] = L.hloc;
            a.meta[4 * ef + 3] = first_head_of_rank(L, a.gpu - rr.dst_g0);
        }
        __syncthreads();
        if (tid == 0) { carry_f += wf[31]; carry_c += wc[31]; }
        __syncthreads();
    }
    const int32_t n_res = carry_f;
    if (tid == 0) a.req_ptr[n_res] = carry_c;
    __syncthreads();
    for (int r = w; r < n_res; r += 32) {
        const int32_t i = a.meta[4 * r];
        const ReqRec rr = a.reqs[i];
        const int32_t start = a.req_ptr[r];
        for (int k = lane; k < rr.n1; k += 32) a.block_ids[start + k] = a.tables[rr.dst_tab + k];
    }
}

cudaError_t launch_remap(const RemapArgs& a, cudaStream_t s) {
    flykv_remap_kernel<<<1, 1024, 0, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- gather
struct GatherArgs {
    GatherSeg seg[3];
    int32_t n_seg;
    char* dst;
};

__global__ void __launch_bounds__(256) flykv_gather_kernel(const GatherArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    int64_t total = 0;
    for (int k = 0; k < a.n_seg; ++k) total += a.seg[k].rows;
    for (int64_t row = warp; row < total; row += nwarps) {
        int k = 0;
        int64_t r = row;
        while (k < a.n_seg - 1 && r >= a.seg[k].rows) { r -= a.seg[k].rows; ++k; }
        const GatherSeg& g = a.seg[k];
        const char* src = g.ptr + r * g.ld_bytes;
        char* dst = a.dst + g.out_off + r * g.row_bytes;
        const bool vec = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) |
                           (uintptr_t)g.row_bytes) & 15) == 0;
        if (vec) {
            for (int64_t i = lane; i < (g.row_bytes >> 4); i += 32)
                reinterpret_cast<int4*>(dst)[i] = __ldg(reinterpret_cast<const int4*>(src) + i);
        } else {
            for (int64_t i = lane; i < g.row_bytes; i += 32) dst[i] = src[i];
        }
    }
}

cudaError_t launch_gather(const GatherSeg* segs, int n_seg, char* dst, cudaStream_t s) {
    GatherArgs a;
    a.n_seg = n_seg;
    a.dst = dst;
    int64_t rows = 0;
    for (int k = 0; k < n_seg && k < 3; ++k) { a.seg[k] = segs[k]; rows += segs[k].rows; }
    int grid = (int)((rows + 7) / 8);
    if (grid > 148 * 8) grid = 148 * 8;
    if (grid < 1) grid = 1;
    flykv_gather_kernel<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

}  // namespace flykv
