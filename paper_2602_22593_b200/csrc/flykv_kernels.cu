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
#include <cstdlib>

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

// One 16-byte store through an NVLS multicast address: NVSwitch writes it to
// every pool bound to the multicast object (the bits are stored as is).
__device__ __forceinline__ void st_multimem(int4* p, const int4& v) {
    asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// Decoded atom: source pointer plus what is needed to form each
// destination replica's pointer (kept in scalars, no local arrays).
struct AtomAddr {
    const char* src;
    int64_t doff;      // byte offset of the atom inside a destination layer region
    int32_t l, h;      // layer, head
    int32_t dst_g0, rep1, hloc1;
    int32_t dst_inv;   // member-of-rank-ID table offset (-1 = identity rank IDs)
    int32_t kv, c;     // K/V half, chunk (kv_pack's send-chunk position)
    int32_t h0, nh, C, k1, J1, a2a;  // segment fields kv_pack needs
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

// Mixed slot (the kernels' atom index) -> piece-space slot, or -1 for a hole
// (MixStream, flykv_internal.h).  MIX = false (launches whose streams are all
// single buckets, a.mixed == 0): the two index spaces coincide and none of
// this is compiled into the kernel.
template <bool MIX>
__device__ __forceinline__ int64_t unmix(const ReshardArgs& a, int64_t atom) {
    if constexpr (!MIX) return atom;
    if (!a.mixed) return atom;
    int lo = a.st_lo, hi = a.st_hi;  // streams[lo].begin <= atom
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (__ldg(&a.streams[mid].begin) <= atom) lo = mid;
        else hi = mid;
    }
    const MixStream ms = a.streams[lo];
    const uint32_t x = (uint32_t)(atom - ms.begin);
    const uint32_t q = x / (uint32_t)ms.Qs, r = x - q * (uint32_t)ms.Qs;
    int b = ms.b0;
    while (b + 1 < ms.b0 + ms.nb && (uint32_t)__ldg(&a.buckets[b + 1].P) <= r) ++b;
    const MixBucket mb = a.buckets[b];
    const int64_t o = (int64_t)q * mb.u + (r - (uint32_t)mb.P);
    return o < mb.size ? mb.start + o : -1;
}

// Slot `local` of the segment at piece-space position s.
template <bool MIX>
__device__ __forceinline__ void decode(const ReshardArgs& a, int s, uint32_t local, AtomAddr& out) {
    const Seg sg = a.segs[MIX && a.mixed ? __ldg(a.seg_of + s) : s];  // plan order: seg_of is the identity
    // destination-major order without holes (Seg, flykv_internal.h): per
    // (layer, K/V) C*nh slots = the destination blocks jb in turn, each nh
    // heads x k1 chunks, the last block nh x kk (kk = C - (J1-1)*k1)
    const uint32_t nh = (uint32_t)sg.nh, k1 = (uint32_t)sg.k1, J1 = (uint32_t)sg.J1, C = (uint32_t)sg.C;
    const uint32_t per = C * nh;
    const uint32_t lkv = local / per;
    uint32_t rem = local - lkv * per;
    const uint32_t row = nh * k1, full = (J1 - 1) * row;
    uint32_t jb, hh, w;
    if (rem < full) {
        jb = rem / row;
        rem -= jb * row;
        hh = rem / k1;
        w = rem - hh * k1;
    } else {
        const uint32_t kk = C - (J1 - 1) * k1;
        rem -= full;
        jb = J1 - 1;
        hh = rem / kk;
        w = rem - hh * kk;
    }
    const uint32_t kv = lkv & 1u, l = lkv >> 1;
    const uint32_t c = jb * k1 + w;
    int32_t h = sg.h0 + (int32_t)hh;
    out.kv = (int32_t)kv;
    out.c = (int32_t)c;
    out.h0 = sg.h0;
    out.nh = sg.nh;
    out.C = sg.C;
    out.k1 = sg.k1;
    out.J1 = sg.J1;
    out.a2a = sg.a2a;
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
    out.dst_inv = sg.dst_inv;
}

// Position of an atom in its (segment, member) run of a send chunk: the
// reshard's destination-major order restricted to the member's nhm heads,
// holes removed -- per (layer, K/V): destination blocks jb, in each the
// member's heads hm, in each chunk w < kk (kk = k1, or what is left of C in
// the last block).  So unpack writes each destination block sequentially.
__device__ __forceinline__ int64_t a2a_pos(int32_t l, int32_t kv, int32_t c, int32_t hm, int32_t nhm, int32_t C,
                                           int32_t k1, int32_t J1) {
    const int32_t jb = c / k1, w = c % k1;
    const int32_t kk = jb == J1 - 1 ? C - jb * k1 : k1;
    return (int64_t)(l * 2 + kv) * nhm * C + (int64_t)jb * nhm * k1 + (int64_t)hm * kk + w;
}

// Pointer to replica j of the decoded atom (1 replica, or p/H under GQA, R2):
// rank ID owning head h, then the member engine holding that rank ID.
__device__ __forceinline__ char* dst_ptr(const ReshardArgs& a, const AtomAddr& ad, int j) {
    const int32_t rid = ad.rep1 == 1 ? ad.h / ad.hloc1 : ad.h * ad.rep1 + j;
    const int32_t m = ad.dst_inv < 0 ? rid : __ldg(a.tables + ad.dst_inv + rid);
    if (a.staged == 3) {  // kv_pack: position in the send chunk of the destination GPU (a2a_pos)
        int32_t first = ad.h, nhm = 1;
        if (ad.rep1 == 1) {
            const int32_t lo = rid * ad.hloc1, hi = lo + ad.hloc1;
            first = lo > ad.h0 ? lo : ad.h0;
            nhm = (hi < ad.h0 + ad.nh ? hi : ad.h0 + ad.nh) - first;
        }
        const int64_t pos = a2a_pos(ad.l, ad.kv, ad.c, ad.h - first, nhm, ad.C, ad.k1, ad.J1);
        return a.a2a_buf + a.a2a_off[ad.dst_g0 + m] + (__ldg(a.a2a_base + ad.a2a + m) + pos) * a.atom_bytes;
    }
    return a.layer_base[(ad.dst_g0 + m) * a.L + ad.l] + ad.doff;
}

// Lane-parallel decode: each lane of the warp decodes one of 32 consecutive
// atoms, then the warp walks them, receiving addresses by shuffle -- the
// index arithmetic costs 1/32 of an issue slot per atom.  Only the source,
// replica-0 destination and replica count stay live; replicas > 0 (GQA)
// re-decode their atom.
struct LaneAtom {
    const char* src;
    char* dst0;
    int32_t rep1;
};

template <bool MIX, bool MC = false>
__device__ __forceinline__ void lane_decode(const ReshardArgs& a, int64_t slot, LaneAtom& la) {
    const int64_t atom = unmix<MIX>(a, slot);
    if (atom < 0) {  // hole of the mixed order
        la.src = nullptr;
        la.dst0 = nullptr;
        la.rep1 = 0;
        return;
    }
    const int s = find_seg(a.seg_begin, a.seg_lo, a.seg_hi, atom);
    const uint32_t local = (uint32_t)(atom - __ldg(a.seg_begin + s));
    AtomAddr ad;
    decode<MIX>(a, s, local, ad);
    la.src = ad.src;
    la.rep1 = ad.rep1;
    la.dst0 = ad.src ? dst_ptr(a, ad, 0) : nullptr;
    if constexpr (MC) {
        // NVLS: the replicas of head h are the team [dst_g0 + h*rep1, +rep1)
        // (identity rank IDs); if this process registered that team, one
        // multimem store (rep1 = -1) replaces the rep1 per-replica stores
        if (ad.rep1 > 1 && ad.dst_inv < 0 && a.staged == 0) {
            const int32_t team = ad.dst_g0 + ad.h * ad.rep1;
            if (__ldg(a.mc_team + team) == ad.rep1) {
                la.dst0 = a.mc_base[(int64_t)team * a.L + ad.l] + ad.doff;
                la.rep1 = -1;
            }
        }
    }
    if ((a.staged == 1 || a.staged == 2) && la.rep1 > 0) {  // comparator: slot-order pack or unpack
        char* stg = a.staging + (slot - a.atom_lo) * (int64_t)a.atom_bytes;
        if (a.staged == 1) {
            la.dst0 = stg;
            la.rep1 = 1;
        } else {
            la.src = stg;
        }
    }
}

template <typename T>
__device__ __forceinline__ T shfl_ptr(T p, int k) {
    return reinterpret_cast<T>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(p), k));
}

// Destination of replica j of the atom at kernel slot `slot` (warp-uniform
// re-decode, GQA replication only; nothing extra is kept live per atom).
template <bool MIX>
__device__ __forceinline__ char* replica_ptr(const ReshardArgs& a, int64_t slot, int j) {
    const int64_t atom = unmix<MIX>(a, slot);
    const int s = find_seg(a.seg_begin, a.seg_lo, a.seg_hi, atom);
    AtomAddr ad;
    decode<MIX>(a, s, (uint32_t)(atom - __ldg(a.seg_begin + s)), ad);
    return dst_ptr(a, ad, j);
}

// ---------------------------------------------------------------- LDG/STG
// VPL = 16-byte vectors per lane per atom (atom_bytes = VPL * 512).  Each
// warp moves one 4 KiB atom per iteration: 8 x LDG.128 per lane issued back
// to back (32 KiB... per warp in flight: 4 KiB), then 8 x STG.128 per
// destination replica.  VPL = 0: generic atoms (multiple of 16 bytes).
// U = atoms per warp iteration: the loads of U atoms (U * 8 LDG.128 per
// lane for 4 KiB atoms) are in flight before their stores are issued.
// Number of steps of round R for this warp (atoms R + k*nwarps + warp < hi).
__device__ __forceinline__ int round_len(const ReshardArgs& a, int64_t R, int64_t warp, int64_t nwarps) {
    const int64_t first = R + warp;
    if (first >= a.atom_hi) return 0;
    const int64_t span = (a.atom_hi - first + nwarps - 1) / nwarps;
    return span < 32 ? (int)span : 32;
}

template <int VPL, int U, bool MIX, bool MC = false>
__global__ void __launch_bounds__(U > 2 ? 128 : 256, U > 2 ? 1 : 2) flykv_reshard_kernel(const ReshardArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    // Round R covers atoms [R, R + 32*nwarps); step k of every warp touches
    // atom R + k*nwarps + warp, so at any moment the whole grid works on one
    // window of nwarps consecutive atoms (~19 MB): few DRAM pages open at
    // once (measured +5-9% over warp-contiguous chunks, scripts/microbench.cu).
    if constexpr (VPL > 0 && U > 1) {
        // Software-pipelined decode: the next round's addresses are decoded
        // right after the first loads of this round are issued, so the
        // decode's dependent-load chain overlaps with bytes in flight.
        int64_t R = a.atom_lo;
        int n = round_len(a, R, warp, nwarps);
        LaneAtom la;
        if (lane < n) lane_decode<MIX, MC>(a, R + warp + lane * nwarps, la);
        while (n > 0) {
            const int64_t first = R + warp;
            const int64_t Rn = R + 32 * nwarps;
            const int nn = round_len(a, Rn, warp, nwarps);
            LaneAtom nx;
            for (int k0 = 0; k0 < n; k0 += U) {
                int4 v[U][VPL];
                const char* s[U];
                char* d0[U];
                int rep[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = (k0 + u < n) ? k0 + u : k0;
                    s[u] = shfl_ptr(la.src, k);
                    d0[u] = shfl_ptr(la.dst0, k);
                    rep[u] = (k0 + u < n) ? __shfl_sync(0xffffffffu, la.rep1, k) : 0;
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (rep[u] == 0) continue;  // hole or past the round (warp-uniform)
                    const int4* src = reinterpret_cast<const int4*>(s[u]) + lane;
#pragma unroll
                    for (int i = 0; i < VPL; ++i) v[u][i] = ld_stream(src + i * 32);
                }
                if (k0 == 0 && lane < nn) lane_decode<MIX, MC>(a, Rn + warp + lane * nwarps, nx);
                // GQA replicas (p > H): lane j decodes replica j's pointer, all
                // replicas of an atom in one parallel pass while its loads are
                // in flight; the stores receive them by shuffle
                const bool par = a.rep_flags & 1;
                char* rp[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    rp[u] = nullptr;
                    if (par && rep[u] > 1 && lane > 0 && lane < rep[u])
                        rp[u] = replica_ptr<MIX>(a, first + (int64_t)(k0 + u) * nwarps, lane);
                }
                auto dst_of = [&](int u, int j) -> int4* {
                    char* dj = j == 0             ? d0[u]
                               : (par && j < 32) ? shfl_ptr(rp[u], j)
                                                 : replica_ptr<MIX>(a, first + (int64_t)(k0 + u) * nwarps, j);
                    return reinterpret_cast<int4*>(dj) + lane;
                };
                if constexpr (MC) {  // NVLS team stores: one (multicast) store per atom
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        if (rep[u] >= 0) continue;
                        int4* dst = reinterpret_cast<int4*>(d0[u]) + lane;
                        if (a.mc_mode == 1) {
#pragma unroll
                            for (int i = 0; i < VPL; ++i) st_multimem(dst + i * 32, v[u][i]);
                        } else {
#pragma unroll
                            for (int i = 0; i < VPL; ++i) st_stream(dst + i * 32, v[u][i]);
                        }
                    }
                }
                if (a.rep_flags & 2) {  // replica-major: replica j of all U atoms, then j + 1
                    int maxr = 0;
#pragma unroll
                    for (int u = 0; u < U; ++u) maxr = rep[u] > maxr ? rep[u] : maxr;
                    for (int j = 0; j < maxr; ++j) {
#pragma unroll
                        for (int u = 0; u < U; ++u) {
                            if (j >= rep[u]) continue;
                            int4* dst = dst_of(u, j);
#pragma unroll
                            for (int i = 0; i < VPL; ++i) st_stream(dst + i * 32, v[u][i]);
                        }
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        for (int j = 0; j < rep[u]; ++j) {
                            int4* dst = dst_of(u, j);
#pragma unroll
                            for (int i = 0; i < VPL; ++i) st_stream(dst + i * 32, v[u][i]);
                        }
                    }
                }
            }
            la = nx;
            R = Rn;
            n = nn;
        }
    } else {
        for (int64_t R = a.atom_lo; R < a.atom_hi; R += 32 * nwarps) {
            const int64_t first = R + warp;
            const int n = round_len(a, R, warp, nwarps);
            if (n == 0) break;
            LaneAtom la;
            if (lane < n) lane_decode<MIX>(a, first + lane * nwarps, la);
            if constexpr (VPL > 0) {
                for (int k = 0; k < n; ++k) {
                    const int4* src = reinterpret_cast<const int4*>(shfl_ptr(la.src, k)) + lane;
                    int4* dst = reinterpret_cast<int4*>(shfl_ptr(la.dst0, k)) + lane;
                    const int rep = __shfl_sync(0xffffffffu, la.rep1, k);
                    if (rep == 0) continue;  // hole (warp-uniform)
                    int4 v[VPL];
#pragma unroll
                    for (int i = 0; i < VPL; ++i) v[i] = ld_stream(src + i * 32);
#pragma unroll
                    for (int i = 0; i < VPL; ++i) st_stream(dst + i * 32, v[i]);
                    for (int j = 1; j < rep; ++j) {
                        int4* dj = reinterpret_cast<int4*>(replica_ptr<MIX>(a, first + k * nwarps, j)) + lane;
#pragma unroll
                        for (int i = 0; i < VPL; ++i) st_stream(dj + i * 32, v[i]);
                    }
                }
            } else {
                for (int k = 0; k < n; ++k) {
                    const char* s = shfl_ptr(la.src, k);
                    char* d0 = shfl_ptr(la.dst0, k);
                    const int rep = __shfl_sync(0xffffffffu, la.rep1, k);
                    const int nv = a.atom_bytes >> 4;
                    for (int j = 0; j < rep; ++j) {
                        char* dj = j == 0 ? d0 : replica_ptr<MIX>(a, first + k * nwarps, j);
                        for (int i = lane; i < nv; i += 32)
                            st_stream(reinterpret_cast<int4*>(dj) + i, ld_stream(reinterpret_cast<const int4*>(s) + i));
                    }
                }
            }
        }
    }
    if (a.fence_sys) __threadfence_system();
}

// ---------------------------------------------------------------- unpack
// kv_unpack: the receiver's side of pack -> all-to-all -> unpack.  Atom i of
// the receiver belongs to pair items[k] (start <= i); its position inside
// that pair (a2a_pos) gives the layer, K/V half, head and chunk, hence the
// destination address in this GPU's pool; the source is
// the chunk received from the segment's source GPU.  Lane-parallel decode as
// in the reshard kernel: lane k decodes step k, the warp copies by shuffle.
__device__ __forceinline__ void unpack_decode(const UnpackArgs& a, int64_t atom, const char*& src, char*& dst) {
    int lo = 0, hi = a.n_items;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (a.items[mid].start <= atom) lo = mid;
        else hi = mid;
    }
    const A2AItem it = a.items[lo];
    const Seg sg = a.segs[it.seg];
    const int64_t local = atom - it.start;
    // invert a2a_pos: (layer, K/V), then destination block, member head, chunk
    const int32_t nhm = it.nhm;
    const int64_t per = (int64_t)nhm * sg.C;
    const int32_t lkv = (int32_t)(local / per);
    const int32_t r = (int32_t)(local % per);
    const int32_t kv = lkv & 1, l = lkv >> 1;
    const int32_t full = (sg.J1 - 1) * nhm * sg.k1;
    int32_t jb, hm, w;
    if (r < full) {
        jb = r / (nhm * sg.k1);
        const int32_t r2 = r % (nhm * sg.k1);
        hm = r2 / sg.k1;
        w = r2 % sg.k1;
    } else {
        jb = sg.J1 - 1;
        const int32_t kk = sg.C - jb * sg.k1, r2 = r - full;
        hm = r2 / kk;
        w = r2 % kk;
    }
    const int32_t c = jb * sg.k1 + w;
    const int32_t h = (sg.rep1 == 1 ? (it.rid * sg.hloc1 > sg.h0 ? it.rid * sg.hloc1 : sg.h0) : it.rid / sg.rep1) + hm;
    const int32_t blk1 = __ldg(a.tables + sg.dst_tab + c / sg.k1);
    dst = a.layer_base[(sg.dst_g0 + it.m) * a.L + l] + (int64_t)blk1 * a.M + kv * (a.M >> 1) +
          (int64_t)((h % sg.hloc1) * sg.k1 + c % sg.k1) * a.atom_bytes;
    src = a.buf + a.off[sg.src_gpu] + (__ldg(a.a2a_base + sg.a2a + it.m) + local) * a.atom_bytes;
}

// VPL = 16-byte vectors per lane per atom (8 for 4 KiB atoms, 0 = generic);
// U = atoms whose loads are in flight before their stores (as in the reshard).
template <int VPL, int U>
__global__ void __launch_bounds__(256) flykv_unpack_kernel(const UnpackArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int nv = a.atom_bytes >> 4;
    for (int64_t R = 0; R < a.n_atoms; R += 32 * nwarps) {
        const int64_t first = R + warp;
        if (first >= a.n_atoms) break;
        const int64_t span = (a.n_atoms - first + nwarps - 1) / nwarps;
        const int n = span < 32 ? (int)span : 32;
        const char* s = nullptr;
        char* d = nullptr;
        if (lane < n) unpack_decode(a, first + lane * nwarps, s, d);
        if constexpr (VPL > 0) {
            for (int k0 = 0; k0 < n; k0 += U) {
                int4 v[U][VPL];
                int4* dk[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int k = k0 + u < n ? k0 + u : k0;
                    const int4* sk = reinterpret_cast<const int4*>(shfl_ptr(s, k)) + lane;
                    dk[u] = k0 + u < n ? reinterpret_cast<int4*>(shfl_ptr(d, k)) + lane : nullptr;
#pragma unroll
                    for (int i = 0; i < VPL; ++i) v[u][i] = ld_stream(sk + i * 32);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (dk[u] == nullptr) continue;  // past the round (warp-uniform)
#pragma unroll
                    for (int i = 0; i < VPL; ++i) st_stream(dk[u] + i * 32, v[u][i]);
                }
            }
        } else {
            for (int k = 0; k < n; ++k) {
                const int4* sk = reinterpret_cast<const int4*>(shfl_ptr(s, k));
                int4* dk = reinterpret_cast<int4*>(shfl_ptr(d, k));
                for (int i = lane; i < nv; i += 32) st_stream(dk + i, ld_stream(sk + i));
            }
        }
    }
}

static int sm_count_of(int device);

cudaError_t launch_unpack(const UnpackArgs& a, int device, cudaStream_t s) {
    if (a.n_atoms <= 0) return cudaSuccess;
    // experiment knob FLYKV_UNPACK_SHAPE: 0 = U2 x 1 CTA/SM, 1 = U1 x 2, 2 = U2 x 2, 3 = U1 x 4.
    // Default 2: its reads stream the receive buffer, so unlike the reshard it
    // wants 12 warps per SM (c2 unpack 6.30 ms vs 8.07 with 6 warps;
    // profiles/r01_a2a_comparator.jsonl).
    static int shape = -1;
    if (shape < 0) {
        const char* e = getenv("FLYKV_UNPACK_SHAPE");
        shape = e ? atoi(e) : 2;
    }
    const int per = shape == 0 ? 1 : shape == 3 ? 4 : 2;
    const bool u2 = shape == 0 || shape == 2;
    const int64_t want = (a.n_atoms + 6 - 1) / 6;  // small transfers: every warp, few atoms each
    const int64_t cap = (int64_t)sm_count_of(device) * per;
    const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
    if (a.atom_bytes == 4096 && u2) flykv_unpack_kernel<8, 2><<<grid, 192, 0, s>>>(a);
    else if (a.atom_bytes == 4096) flykv_unpack_kernel<8, 1><<<grid, 192, 0, s>>>(a);
    else if (a.atom_bytes == 2048) flykv_unpack_kernel<4, 2><<<grid, 192, 0, s>>>(a);
    else flykv_unpack_kernel<0, 1><<<grid, 192, 0, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- TMA bulk
// Each warp runs its own S-stage shared-memory ring.  Lane 0 drives the
// loads: cp.async.bulk global->shared, completing on a per-stage mbarrier.
// The stores are warp-wide: once a stage's bytes have landed, lane j issues
// the cp.async.bulk shared->global of replica j (1, or p/H under GQA
// replication, R2) from that one stage -- the replicas' address decodes and
// bulk stores run in parallel instead of one after another on lane 0 -- and
// every lane commits one bulk group per atom (empty when it has no replica),
// so the lanes' group sequences stay aligned.  Loads run D = S - 2 atoms
// ahead of the stores; a stage is refilled once every lane's
// cp.async.bulk.wait_group.read shows the stores reading it have finished.
// No data passes through registers.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

template <int S, int W>
__global__ void __launch_bounds__(W * 32) flykv_reshard_tma_kernel(const ReshardArgs a, int stage_bytes) {
    constexpr int D = S - 2;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    unsigned char* ring = smem + (size_t)wid * S * stage_bytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)W * S * stage_bytes) + wid * S;
    // per-stage pending store: replica-0 destination, replica count, atom index (written by lane 0)
    __shared__ char* pend_dst[W][S];
    __shared__ int32_t pend_rep[W][S];
    __shared__ int64_t pend_atom[W][S];
    if (lane == 0) {
        for (int i = 0; i < S; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + i)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    const uint32_t bytes = (uint32_t)a.atom_bytes;
    const int64_t warp = (int64_t)blockIdx.x * W + wid;
    const int64_t nwarps = (int64_t)gridDim.x * W;
    uint32_t issued = 0, stored = 0;  // warp-uniform
    auto store_one = [&](uint32_t j) {  // warp-wide: lane r stores replica r
        const int st = j % S;
        mbar_wait(smem_u32(bars + st), (j / S) & 1u);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t src = smem_u32(ring + (size_t)st * stage_bytes);
        const int rep = pend_rep[wid][st];
        for (int r = lane; r < rep; r += 32) {
            char* dst = r == 0 ? pend_dst[wid][st] : replica_ptr<true>(a, pend_atom[wid][st], r);
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                         "r"(src), "r"(bytes), "l"(policy)
                         : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    };
    // grid-interleaved like the LDG kernel: step k of round R is atom
    // R + k*nwarps + warp, so the grid sweeps one window of consecutive atoms
    for (int64_t R = a.atom_lo; R < a.atom_hi; R += 32 * nwarps) {
        const int n = round_len(a, R, warp, nwarps);
        if (n == 0) break;
        LaneAtom la;
        if (lane < n) lane_decode<true>(a, R + warp + lane * nwarps, la);
        for (int k = 0; k < n; ++k) {
            const char* s = shfl_ptr(la.src, k);
            char* d0 = shfl_ptr(la.dst0, k);
            const int rep = __shfl_sync(0xffffffffu, la.rep1, k);
            if (rep == 0) continue;  // hole (warp-uniform)
            if (issued >= (uint32_t)D) store_one(stored++);
            const int st = issued % S;
            // stage st last held atom issued - S; after the store above, the
            // S - D most recent bulk groups of every lane are atoms
            // issued-S+1 .. issued-D, so waiting down to S - D pending frees it
            asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(S - D) : "memory");
            __syncwarp();
            if (lane == 0) {
                pend_dst[wid][st] = d0;
                pend_rep[wid][st] = rep;
                pend_atom[wid][st] = R + warp + (int64_t)k * nwarps;
                const uint32_t bar = smem_u32(bars + st);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
                    "[%3], %4;" ::"r"(smem_u32(ring + (size_t)st * stage_bytes)),
                    "l"(s), "r"(bytes), "r"(bar), "l"(policy)
                    : "memory");
            }
            __syncwarp();
            ++issued;
        }
    }
    while (stored < issued) store_one(stored++);
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    if (a.fence_sys) __threadfence_system();
    __syncwarp();
}

// ---------------------------------------------------------------- launch
static int g_impl = 0;          // 0 auto, 1 LDG, 2 TMA
static int g_ctas_per_sm = 0;   // 0 auto
static int g_threads = 0;       // threads per CTA of the LDG kernel, 0 = default (experiment knob: FLYKV_THREADS)

static int g_rep_flags = -1;    // replica store strategy (ReshardArgs::rep_flags), -1 = default

// Experiment knobs (launch shape and replica strategy sweeps, scripts/): read
// once from the environment; the defaults are the measured optima.
static void read_env_knobs() {
    static bool done = false;
    if (done) return;
    done = true;
    const char* t = getenv("FLYKV_THREADS");
    if (t && atoi(t) >= 32 && atoi(t) <= 256 && atoi(t) % 32 == 0) g_threads = atoi(t);
    const char* c = getenv("FLYKV_CTAS");
    if (c && atoi(c) >= 1 && atoi(c) <= 8) g_ctas_per_sm = atoi(c);
    const char* r = getenv("FLYKV_REP_FLAGS");
    if (r && atoi(r) >= 0 && atoi(r) <= 3) g_rep_flags = atoi(r);
}

void set_reshard_impl(int impl, int ctas_per_sm) {
    read_env_knobs();
    g_impl = impl;
    g_ctas_per_sm = ctas_per_sm;
}

static int sm_count_of(int device) {
    static int cache[64] = {0};
    if (device < 0 || device >= 64) device = 0;
    if (cache[device] == 0) cudaDeviceGetAttribute(&cache[device], cudaDevAttrMultiProcessorCount, device);
    return cache[device] > 0 ? cache[device] : 148;
}

template <int VPL, int U = 1>
static cudaError_t launch_ldg(const ReshardArgs& a_in, int device, cudaStream_t s) {
    read_env_knobs();
    ReshardArgs a = a_in;
    // Replica stores (GQA): 2-3 replicas: serial re-decode, replica-major
    // (rep_flags 2) at 7 warps per SM (H_kv=4 -> TP8 forward 11.77 ms
    // against 11.96 for lane-parallel decode at 6 warps, round 2,
    // profiles/r02_gqa_replica_sweep.txt); 4-7 replicas (peer destinations;
    // local ones take the TMA ring): lane-parallel decode; 8+: serial
    // re-decode between replica stores, which spaces the store bursts
    // (round 1, profiles/r01_gqa_rep.jsonl).
    a.rep_flags = g_rep_flags >= 0 ? g_rep_flags : (a.max_rep > 1 && a.max_rep < 4 ? 2 : a.max_rep < 8 ? 1 : 0);
    static int per_sm = 0;
    if (per_sm == 0) {
        int nb = 0;
        cudaError_t e =
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, flykv_reshard_kernel<VPL, U, false>, U > 2 ? 128 : 256, 0);
        if (e != cudaSuccess) return e;
        per_sm = nb > 0 ? nb : 1;
    }
    const int64_t atoms = a.atom_hi - a.atom_lo;
    // Bytes in flight per SM are the tuning parameter: more concurrent
    // streams cost DRAM row locality, fewer starve the memory system.  The
    // measured optimum is 6 warps x 8 KiB = 48 KiB per SM (U=2: one 192-thread
    // CTA per SM: 6.45-6.59 TB/s on C2/C4, vs 6.26-6.30 with 8 warps and
    // 5.9 with 4; scripts/variants.py).  U=1: two 256-thread CTAs.
    // GQA replication (p/H copies per read) is write-heavy: on this path
    // (peer destinations, or FLYKV_REP_TMA=0) 8 replicas want 10 warps per
    // SM (2 x 160 threads; round 1: H_kv=1 TP8 5.55 ms vs 5.73-7.2 for other
    // shapes); 2-3 replicas with replica-major stores want 7 (224 threads).
    int want_per = U == 1 ? 2 : 1, want_threads = U == 1 ? 256 : U == 2 ? 192 : U == 3 ? 128 : 96;
    if (U == 2 && a.max_rep >= 8) {
        want_threads = 160;
        want_per = 2;
    } else if (U == 2 && a.max_rep > 1 && a.max_rep < 4) {
        want_threads = 224;  // 7 warps with the replica-major stores (above)
    }
    const int per = g_ctas_per_sm > 0 ? g_ctas_per_sm : (per_sm < want_per ? per_sm : want_per);
    const int threads = g_threads > 0 ? g_threads : want_threads;
    // small plans: spread the atoms over every warp the grid can hold (one
    // or a few atoms per warp) rather than 32 per warp on fewer CTAs -- a
    // warp walks its atoms one after another, so latency, not bandwidth,
    // bounds a switch of a few MB (the tiny config's 4 MiB took 27 us)
    int64_t want = (atoms + (threads / 32) - 1) / (threads / 32);
    int64_t cap = (int64_t)sm_count_of(device) * per;
    int grid = (int)(want < cap ? want : cap);
    if (grid < 1) grid = 1;
    if constexpr (VPL > 0 && U > 1) {  // NVLS team stores (kv_cache_set_multicast)
        if (a.mc_mode) {
            if (a.mixed) flykv_reshard_kernel<VPL, U, true, true><<<grid, threads, 0, s>>>(a);
            else flykv_reshard_kernel<VPL, U, false, true><<<grid, threads, 0, s>>>(a);
            return cudaGetLastError();
        }
    }
    if (a.mixed) flykv_reshard_kernel<VPL, U, true><<<grid, threads, 0, s>>>(a);
    else flykv_reshard_kernel<VPL, U, false><<<grid, threads, 0, s>>>(a);
    return cudaGetLastError();
}

template <int S, int W>
static cudaError_t launch_tma(const ReshardArgs& a, int device, cudaStream_t s, int want_per = 0) {
    const int stage = (a.atom_bytes + 127) & ~127;
    const size_t smem = (size_t)W * S * stage + (size_t)W * S * 8;
    static size_t configured = 0;
    if (smem > configured) {
        cudaError_t e = cudaFuncSetAttribute(flykv_reshard_tma_kernel<S, W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured = smem;
    }
    int per = g_ctas_per_sm > 0 ? g_ctas_per_sm : want_per;
    int nb = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, flykv_reshard_tma_kernel<S, W>, W * 32, smem);
    if (e != cudaSuccess) return e;
    if (per <= 0 || per > nb) per = nb > 0 ? nb : 1;
    const int64_t atoms = a.atom_hi - a.atom_lo;
    int64_t want = (atoms + W - 1) / W;  // small plans: every warp, few atoms each
    int64_t cap = (int64_t)sm_count_of(device) * per;
    int grid = (int)(want < cap ? want : cap);
    if (grid < 1) grid = 1;
    flykv_reshard_tma_kernel<S, W><<<grid, W * 32, smem, s>>>(a, stage);
    return cudaGetLastError();
}

// TMA ring shape (stages x warps per CTA), experiment knob FLYKV_TMA_SHAPE.
// Default: 4 stages x 2 warps x 3 CTAs per SM = 6 warps with 2 loads ahead
// each -- 48 KiB in flight per SM, the same optimum as the LDG kernel
// (c2: 6.36 TB/s vs 4.9 for 8 stages x 4 warps; profiles/r01_tma.jsonl).
static cudaError_t launch_tma_shape(const ReshardArgs& a, int device, cudaStream_t s) {
    static int shape = -1;
    if (shape < 0) {
        const char* e = getenv("FLYKV_TMA_SHAPE");
        shape = e ? atoi(e) : 0;
    }
    switch (shape) {
        case 1: return launch_tma<4, 4>(a, device, s);
        case 3: return launch_tma<6, 2>(a, device, s);
        case 4: return launch_tma<8, 2>(a, device, s);
        case 5: return launch_tma<4, 8>(a, device, s);
        case 6: return launch_tma<3, 4>(a, device, s);
        case 7: return launch_tma<6, 4>(a, device, s);
        case 8: return launch_tma<3, 8>(a, device, s);
        case 9: return launch_tma<8, 4>(a, device, s);
        case 10: return launch_tma<4, 1>(a, device, s);
        case 11: return launch_tma<6, 1>(a, device, s);
        case 12: return launch_tma<8, 1>(a, device, s);
        case 13: return launch_tma<3, 2>(a, device, s);
        case 14: return launch_tma<5, 2>(a, device, s);
        case 15: return launch_tma<4, 3>(a, device, s);
        case 16: return launch_tma<3, 1>(a, device, s);
        case 17: return launch_tma<12, 1>(a, device, s);
        default: return launch_tma<4, 2>(a, device, s, 3);
    }
}

cudaError_t launch_reshard(const ReshardArgs& a, int device, cudaStream_t s) {
    if (a.atom_hi <= a.atom_lo) return cudaSuccess;
    const bool tma_ok = (a.atom_bytes % 16) == 0 && a.atom_bytes <= 16384;
    if (g_impl == 2 && tma_ok && !a.peer && !a.mc_mode) return launch_tma_shape(a, device, s);
    // GQA replication with >= 4 replicas (p/H, R2) into local pools: most of
    // the traffic is writes, and the TMA ring with lane-parallel replica bulk
    // stores writes them fastest -- the more replicas, the fewer loads in
    // flight it wants: 8 replicas at 2 warps per SM (2 CTAs x 1 warp, 4
    // stages, 2 atoms ahead; H_kv=1 -> TP8 forward 8.82 ms against 9.22 ms
    // for the best LDG/STG shape), 4 replicas at 6 warps per SM (6 CTAs x 1
    // warp, 3 stages, 1 atom ahead; H_kv=2 forward 9.80 ms against 10.22 for
    // the best LDG/STG shape and 10.57 for the round-1 default).  Sweeps:
    // profiles/r02_gqa_tma*.jsonl, r02_gqa_replica_sweep.txt.  Knob
    // FLYKV_REP_TMA=0 keeps the LDG/STG kernel (A/B).
    static int rep_tma = -1;
    if (rep_tma < 0) {
        const char* e = getenv("FLYKV_REP_TMA");
        rep_tma = e ? atoi(e) : 1;
    }
    if (g_impl == 0 && rep_tma && a.max_rep >= 4 && tma_ok && !a.peer && !a.mc_mode && a.staged != 1 && a.staged != 2)
        return a.max_rep >= 8 ? launch_tma<4, 1>(a, device, s, 2) : launch_tma<3, 1>(a, device, s, 6);
    // default (0) and 3: two atoms in flight per warp (measured +1%)
    // experiment knob FLYKV_U: atoms in flight per warp for 4 KiB atoms (2 default; 3, 4)
    static int u_knob = -1;
    if (u_knob < 0) {
        const char* e = getenv("FLYKV_U");
        u_knob = e ? atoi(e) : 2;
    }
    if ((g_impl == 0 || g_impl == 3) && a.atom_bytes == 4096 && u_knob == 3) return launch_ldg<8, 3>(a, device, s);
    if ((g_impl == 0 || g_impl == 3) && a.atom_bytes == 4096 && u_knob == 4) return launch_ldg<8, 4>(a, device, s);
    if ((g_impl == 0 || g_impl == 3) && a.atom_bytes == 4096) return launch_ldg<8, 2>(a, device, s);
    if ((g_impl == 0 || g_impl == 3) && a.atom_bytes == 2048) return launch_ldg<4, 2>(a, device, s);
    switch (a.atom_bytes) {
        case 512: return launch_ldg<1>(a, device, s);
        case 1024: return launch_ldg<2>(a, device, s);
        case 2048: return launch_ldg<4>(a, device, s);
        case 4096: return launch_ldg<8>(a, device, s);
        case 8192: return launch_ldg<16>(a, device, s);
        default: return launch_ldg<0>(a, device, s);
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
    // all-GPU mode: CTA g writes pool g's table into its slice of packed outputs
    const int32_t gpu = a.out_off ? (int32_t)blockIdx.x : a.gpu;
    int32_t* req_ptr = a.req_ptr + (a.out_off ? a.out_off[3 * gpu + 0] : 0);
    int32_t* block_ids = a.block_ids + (a.out_off ? a.out_off[3 * gpu + 1] : 0);
    int32_t* meta = a.meta + (a.out_off ? a.out_off[3 * gpu + 2] : 0);
    if (tid == 0) { carry_f = 0; carry_c = 0; }
    __syncthreads();
    for (int base = 0; base < a.n_reqs; base += 1024) {
        const int i = base + tid;
        int32_t flag = 0, cnt = 0;
        ReqRec rr = {0, 1, 0, 0};
        if (i < a.n_reqs) {
            rr = a.reqs[i];
            flag = (gpu >= rr.dst_g0 && gpu < rr.dst_g0 + rr.dst_p) ? 1 : 0;
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
            req_ptr[ef] = ec;
            meta[4 * ef + 0] = i;
            meta[4 * ef + 1] = a.B * L.k;
            meta[4 * ef + 2] = L.hloc;
            const int32_t m = gpu - rr.dst_g0;
            meta[4 * ef + 3] = first_head_of_rank(L, rr.dst_rid < 0 ? m : a.tables[rr.dst_rid + m]);
        }
        __syncthreads();
        if (tid == 0) { carry_f += wf[31]; carry_c += wc[31]; }
        __syncthreads();
    }
    const int32_t n_res = carry_f;
    if (tid == 0) req_ptr[n_res] = carry_c;
    __syncthreads();
    for (int r = w; r < n_res; r += 32) {
        const int32_t i = meta[4 * r];
        const ReqRec rr = a.reqs[i];
        const int32_t start = req_ptr[r];
        for (int k = lane; k < rr.n1; k += 32) block_ids[start + k] = a.tables[rr.dst_tab + k];
    }
}

cudaError_t launch_remap(const RemapArgs& a, int n_ctas, cudaStream_t s) {
    flykv_remap_kernel<<<n_ctas, 1024, 0, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- barrier
// a5, group completion barrier between processes (one per GPU, "safe
// points"): one thread.  Every earlier kernel of this stream (the reshard,
// whose peer stores end with a system-scope fence) has completed; the
// sequentially consistent system fence orders them before the arrivals.
// Arrive: a system-scope release add of 1 to every member's counter
// (including this process's own).  Wait: acquire loads of the own counter
// until it reaches `target` = (barriers so far on this counter) x members:
// every member then has arrived (each adds exactly once per barrier and
// none can pass barrier k+1 before all have arrived at it).  A member that
// never arrives ends the wait after timeout_ns (%globaltimer): *status = 1
// if status is given, else the kernel traps (a loud CUDA error, never a hang).
__device__ __forceinline__ bool group_barrier(unsigned long long* const* flags, int n, int self, uint64_t target,
                                              int64_t timeout_ns) {
    asm volatile("fence.sc.sys;" ::: "memory");
    for (int m = 0; m < n; ++m) asm volatile("red.release.sys.global.add.u64 [%0], 1;" ::"l"(flags[m]) : "memory");
    uint64_t t0, t, v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (true) {
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags[self]) : "memory");
        if (v >= target) return true;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if ((int64_t)(t - t0) > timeout_ns) return false;
        __nanosleep(200);
    }
}

__global__ void flykv_barrier_kernel(const BarrierArgs a) {
    if (group_barrier(a.flags, a.n, a.self, a.target, a.timeout_ns)) return;
    if (a.status) {
        *a.status = 1;
        return;
    }
    __trap();
}

cudaError_t launch_barrier(const BarrierArgs& a, cudaStream_t s) {
    flykv_barrier_kernel<<<1, 1, 0, s>>>(a);
    return cudaGetLastError();
}

// kv_group_barrier_selftest: the members of one group emulated as the CTAs of
// ONE cooperative launch (co-resident by construction -- separate launches
// that spin on one another are never run on one device).  CTA m is member m:
// per round k it stores k into its payload word (its "push"), runs the
// production barrier (group_barrier, target k*n on its own counter), then
// loads every member's payload: a value < k means a member passed the
// barrier before another's push was visible.  CTA `absent` never arrives
// (timeout path).  counters: n lines of 16 u64; payload: n lines of 16 u64.
__global__ void flykv_barrier_selftest_kernel(const BarrierArgs a, int32_t rounds, int32_t absent,
                                              unsigned long long* payload, int32_t* errors, int32_t* timeouts) {
    const int m = blockIdx.x;
    if (threadIdx.x != 0 || m == absent) return;
    for (int32_t k = 1; k <= rounds; ++k) {
        volatile unsigned long long* mine = payload + 16 * m;
        *mine = (unsigned long long)k;
        if (!group_barrier(a.flags, a.n, m, (uint64_t)k * a.n, a.timeout_ns)) {
            atomicAdd(timeouts, 1);
            return;
        }
        for (int j = 0; j < a.n; ++j) {
            const volatile unsigned long long* other = payload + 16 * j;
            if (*other < (unsigned long long)k) atomicAdd(errors, 1);
        }
    }
}

cudaError_t launch_barrier_selftest(const BarrierArgs& a, int32_t rounds, int32_t absent,
                                    unsigned long long* payload, int32_t* errors, int32_t* timeouts, cudaStream_t s) {
    BarrierArgs aa = a;
    void* args[] = {&aa, &rounds, &absent, &payload, &errors, &timeouts};
    return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(flykv_barrier_selftest_kernel), dim3(a.n), dim3(32),
                                       args, 0, s);
}

// ---------------------------------------------------------------- verify
// R10 strict mode: CTA (item, layer*2 + kv), one warp per chunk.  Under
// replication (p0 > H) H_loc = 1, so chunk c of the head is at block
// tab[c / k0], offset kv*M/2 + (c % k0) * atom in both replicas (uniform
// IDs, R6).  Only the valid tokens of the last chunk are compared.
__global__ void __launch_bounds__(256) flykv_verify_kernel(const VerifyArgs a) {
    const ReplicaItem it = a.items[blockIdx.x];
    const int32_t l = blockIdx.y >> 1, kv = blockIdx.y & 1;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int32_t c = wid; c < it.C; c += nw) {
        const int32_t blk = __ldg(a.tables + it.src_tab + c / it.k0);
        const int64_t off = (int64_t)blk * a.M + kv * (a.M >> 1) + (int64_t)(c % it.k0) * a.atom_bytes;
        const char* x = a.layer_base[it.gpu_c * a.L + l] + off;
        const char* y = a.layer_base[it.gpu_r * a.L + l] + off;
        const int64_t tok = (c == it.C - 1) ? (int64_t)it.T - (int64_t)c * a.B : a.B;
        const int64_t nbytes = tok * a.tok_bytes;
        bool diff = false;
        for (int64_t i = (int64_t)lane * 16; i + 16 <= nbytes; i += 32 * 16) {
            const int4 u = ld_stream(reinterpret_cast<const int4*>(x + i));
            const int4 v = ld_stream(reinterpret_cast<const int4*>(y + i));
            diff |= (u.x != v.x) | (u.y != v.y) | (u.z != v.z) | (u.w != v.w);
        }
        for (int64_t i = (nbytes & ~(int64_t)15) + lane; i < nbytes; i += 32) diff |= x[i] != y[i];
        if (__any_sync(0xffffffffu, diff) && lane == 0) {
            atomicAdd(a.out, 1ull);
            const unsigned long long code =
                ((unsigned long long)((int64_t)blockIdx.x * 2 * a.L + blockIdx.y) << 32) | (unsigned)c;
            atomicMin(a.out + 1, code);
        }
    }
}

cudaError_t launch_verify(const VerifyArgs& a, cudaStream_t s) {
    if (a.n_items <= 0) return cudaSuccess;
    dim3 grid((unsigned)a.n_items, (unsigned)(2 * a.L));
    flykv_verify_kernel<<<grid, 256, 0, s>>>(a);
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
