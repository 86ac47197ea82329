// flykv_decode.cu -- consumer proof: paged decode attention
// that reads a pool through the per-request "stride and capacity" the KV Cache
// Adaptor hands to the attention kernel: the CSR block table of
// kv_remap_block_tables and, per request, B(p), H_loc(p) and the first KV head.
//
// One warp per (resident request, local query head).  Lanes hold d/32
// contiguous elements of q, k, v; tokens are visited in order 0..T-1 with an
// fp32 online softmax, and the dot product is reduced by a fixed xor-shuffle
// tree.  The arithmetic therefore depends only on token order, never on the
// block size: a TP rank reading the re-laid-out cache produces bit-for-bit
// the output the DP replica produces for the same heads, which is what the
// test checks.  (A consumer proof, not a tuned attention kernel: the decode
// GEMV is HBM-bound and not on the switch's hot path.)
#include <cuda_bf16.h>

#include "flykv_internal.h"

namespace flykv {

template <int EPL>  // bf16 elements per lane = d / 32
__global__ void __launch_bounds__(128) flykv_paged_decode_kernel(const DecodeArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t item = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (item >= (int64_t)a.n_res * a.q_local) return;
    const int r = (int)(item / a.q_local);
    const int j = (int)(item % a.q_local);
    const int32_t Bp = a.meta[4 * r + 1];
    const int32_t hloc = a.meta[4 * r + 2];
    const int32_t hl = j / (a.q_local / hloc);  // local KV head serving local query head j
    const int32_t T = a.seq_lens[r];
    const int32_t* tab = a.block_ids + a.req_ptr[r];
    const int64_t row = (int64_t)a.d * 2;       // bytes of one token of one head (bf16)
    const int64_t half = a.M >> 1;

    float q[EPL], acc[EPL];
    const __nv_bfloat16* qp = a.q + ((int64_t)r * a.q_local + j) * a.d + lane * EPL;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        q[e] = __bfloat162float(qp[e]);
        acc[e] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    for (int32_t t = 0; t < T; ++t) {
        const int64_t off = (int64_t)tab[t / Bp] * a.M + ((int64_t)hl * Bp + t % Bp) * row + lane * EPL * 2;
        const __nv_bfloat16* kp = reinterpret_cast<const __nv_bfloat16*>(a.layer + off);
        const __nv_bfloat16* vp = reinterpret_cast<const __nv_bfloat16*>(a.layer + off + half);
        float dot = 0.f;
#pragma unroll
        for (int e = 0; e < EPL; ++e) dot = fmaf(q[e], __bfloat162float(kp[e]), dot);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
        const float s = dot * a.scale;
        const float m_new = fmaxf(m, s);
        const float corr = __expf(m - m_new);
        const float p = __expf(s - m_new);
        l = l * corr + p;
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[e] = fmaf(p, __bfloat162float(vp[e]), acc[e] * corr);
        m = m_new;
    }
    float* op = a.out + ((int64_t)r * a.q_local + j) * a.d + lane * EPL;
    const float inv = T > 0 ? 1.f / l : 0.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) op[e] = acc[e] * inv;
}

cudaError_t launch_decode(const DecodeArgs& a, cudaStream_t s) {
    const int64_t warps = (int64_t)a.n_res * a.q_local;
    if (warps == 0) return cudaSuccess;
    const int grid = (int)((warps + 3) / 4);
    switch (a.d) {
        case 64: flykv_paged_decode_kernel<2><<<grid, 128, 0, s>>>(a); break;
        case 128: flykv_paged_decode_kernel<4><<<grid, 128, 0, s>>>(a); break;
        case 256: flykv_paged_decode_kernel<8><<<grid, 128, 0, s>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace flykv
