// microbench_wr.cu -- which write pattern reaches cudaMemset's write bandwidth?
// Write-only variants over 16 GiB: memset-style thread grid-stride, warp per
// 4 KiB atom (the reshard's structure), CTA per 64 KiB chunk, and TMA bulk
// shared->global stores.  Then the same patterns with R=8 replication reads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbwr microbench_wr.cu
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void st4(char* p, int4 v) {
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ void st4_plain(char* p, int4 v) { *reinterpret_cast<int4*>(p) = v; }
__device__ __forceinline__ int4 ld4(const char* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

// (1) memset style: thread t writes 16 B at (i*nthreads + t)*16
template <int PLAIN>
__global__ void w_grid(char* dst, long n16) {
    long t = (long)blockIdx.x * blockDim.x + threadIdx.x, nt = (long)gridDim.x * blockDim.x;
    int4 v = make_int4(1, 2, 3, (int)t);
    for (long i = t; i < n16; i += nt) {
        if (PLAIN) st4_plain(dst + i * 16, v); else st4(dst + i * 16, v);
    }
}
// (1b) memset style with 4 stores per thread per iteration (ILP)
__global__ void w_grid4(char* dst, long n16) {
    long t = (long)blockIdx.x * blockDim.x + threadIdx.x, nt = (long)gridDim.x * blockDim.x;
    int4 v = make_int4(1, 2, 3, (int)t);
    for (long i = t; i < n16; i += 4 * nt) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (i + k * nt < n16) st4(dst + (i + k * nt) * 16, v);
    }
}
// (2) warp per 4 KiB atom, atoms grid-interleaved (atom = round*nwarps + warp)
__global__ void w_warp_atom(char* dst, long natoms) {
    const int lane = threadIdx.x & 31;
    long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
    int4 v = make_int4(1, 2, 3, lane);
    for (long a = warp; a < natoms; a += nw) {
#pragma unroll
        for (int i = 0; i < 8; ++i) st4(dst + a * 4096 + (i * 32 + lane) * 16, v);
    }
}
// (3) warp per atom but instruction-interleaved across the grid: at step i
// warp w writes the i-th 512 B line of atom a -- same as (2); variant: the
// warp's 8 stores go to 8 consecutive atoms' same line? no -- (3) is CTA per
// 64 KiB chunk: the whole CTA writes one chunk coalesced, chunks grid-strided.
__global__ void w_cta_chunk(char* dst, long nchunks) {
    int4 v = make_int4(1, 2, 3, threadIdx.x);
    for (long c = blockIdx.x; c < nchunks; c += gridDim.x) {
        char* base = dst + c * 65536;
        for (int o = threadIdx.x * 16; o < 65536; o += blockDim.x * 16) st4(base + o, v);
    }
}
// (4) TMA bulk store: each warp's lane 0 issues cp.async.bulk S->G of 4 KiB atoms
__global__ void w_bulk(char* dst, long natoms, int max_pending) {
    __shared__ __align__(128) char buf[4096];
    for (int o = threadIdx.x * 16; o < 4096; o += blockDim.x * 16) *reinterpret_cast<int4*>(buf + o) = make_int4(1, 2, 3, o);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const int lane = threadIdx.x & 31;
    long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
    if (lane == 0) {
        uint32_t s = (uint32_t)__cvta_generic_to_shared(buf);
        int pend = 0;
        for (long a = warp; a < natoms; a += nw) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;" ::"l"(dst + a * 4096), "r"(s) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (++pend >= max_pending) {
                asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
                pend = 8;
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}
// (5) R-replicate with memset-style addressing: thread t reads 16 B of source at
// i and writes it to R regions at i (i grid-strided over the source)
__global__ void rep_grid(const char* src, char* dst, long n16_src, int R) {
    long t = (long)blockIdx.x * blockDim.x + threadIdx.x, nt = (long)gridDim.x * blockDim.x;
    for (long i = t; i < n16_src; i += 2 * nt) {
        int4 v0 = ld4(src + i * 16);
        int4 v1 = i + nt < n16_src ? ld4(src + (i + nt) * 16) : v0;
        for (int r = 0; r < R; ++r) {
            st4(dst + ((long)r * n16_src + i) * 16, v0);
            if (i + nt < n16_src) st4(dst + ((long)r * n16_src + i + nt) * 16, v1);
        }
    }
}
// (6) R-replicate, warp per atom (reshard structure), U=2
__global__ void rep_warp(const char* src, char* dst, long n_src, int R) {
    const int lane = threadIdx.x & 31;
    long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
    for (long a0 = warp * 2; a0 < n_src; a0 += nw * 2) {
        int4 v[2][8];
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int i = 0; i < 8; ++i) v[u][i] = ld4(src + min(a0 + u, n_src - 1) * 4096 + (i * 32 + lane) * 16);
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int u = 0; u < 2; ++u)
                if (a0 + u < n_src)
#pragma unroll
                    for (int i = 0; i < 8; ++i) st4(dst + ((long)r * n_src + a0 + u) * 4096 + (i * 32 + lane) * 16, v[u][i]);
    }
}

int main() {
    const long bytes = 16L << 30;
    char *a, *b;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMemset(a, 1, bytes);
    cudaMemset(b, 2, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](auto fn, const char* name, double traffic) {
        for (int i = 0; i < 3; ++i) fn();
        cudaDeviceSynchronize();
        float best = 1e9, sum = 0;
        for (int i = 0; i < 10; ++i) {
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
            sum += ms;
        }
        printf("%-52s best %8.3f ms %7.1f GB/s  mean %7.1f GB/s\n", name, best, traffic / best / 1e6, traffic / (sum / 10) / 1e6);
    };
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    char name[128];
    const long n16 = bytes / 16, natoms = bytes / 4096;
    time([&] { cudaMemsetAsync(b, 3, bytes); }, "cudaMemset", (double)bytes);
    for (int per : {1, 2, 4, 8, 16}) {
        for (int thr : {256, 512, 1024}) {
            if (per * thr > 2048) continue;
            snprintf(name, 128, "grid-stride st %d x %d", sms * per, thr);
            time([&] { w_grid<0><<<sms * per, thr>>>(b, n16); }, name, (double)bytes);
        }
    }
    time([&] { w_grid<1><<<sms * 8, 256>>>(b, n16); }, "grid-stride plain st 8/SM x 256", (double)bytes);
    time([&] { w_grid4<<<sms * 4, 512>>>(b, n16); }, "grid-stride ILP4 4/SM x 512", (double)bytes);
    time([&] { w_grid4<<<sms, 512>>>(b, n16); }, "grid-stride ILP4 1/SM x 512", (double)bytes);
    time([&] { w_grid<0><<<(int)((n16 + 255) / 256), 256>>>(b, n16); }, "one thread per 16 B (non-persistent)", (double)bytes);
    for (int warps : {6, 8, 16, 32}) {
        snprintf(name, 128, "warp per atom, %d warps/SM", warps);
        time([&] { w_warp_atom<<<sms, 32 * warps>>>(b, natoms); }, name, (double)bytes);
    }
    for (int thr : {256, 512, 1024}) {
        snprintf(name, 128, "CTA per 64 KiB chunk, %d x %d", sms * 2048 / thr, thr);
        time([&] { w_cta_chunk<<<sms * 2048 / thr, thr>>>(b, bytes / 65536); }, name, (double)bytes);
    }
    for (int warps : {4, 8, 16}) {
        for (int pend : {16, 32}) {
            snprintf(name, 128, "TMA bulk S->G 4 KiB, %d warps/SM, %d pending", warps, pend);
            time([&] { w_bulk<<<sms, 32 * warps>>>(b, natoms, pend); }, name, (double)bytes);
        }
    }
    for (int R : {1, 8}) {
        double traffic = (double)bytes * (1.0 + 1.0 / R);
        for (int per : {2, 4, 8}) {
            snprintf(name, 128, "rep R=%d grid-stride %d/SM x 256", R, per);
            time([&] { rep_grid<<<sms * per, 256>>>(a, b, n16 / R, R); }, name, traffic);
        }
        for (int warps : {6, 10}) {
            snprintf(name, 128, "rep R=%d warp per atom %d warps/SM", R, warps);
            time([&] { rep_warp<<<sms, 32 * warps>>>(a, b, natoms / R, R); }, name, traffic);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
