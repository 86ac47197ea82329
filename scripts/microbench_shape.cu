// microbench_shape.cu -- copy structure vs DRAM efficiency for the
// re-layout's pattern: 64 KiB blocks in a seeded random permutation on both
// sides (the pools' scattered blocks), 16 GiB moved, 80 GiB footprints.
//   A  warp per 4 KiB atom, grid-interleaved, U atoms in flight per warp
//   B  CTA per 64 KiB block (each thread 16 x 16 B per block), grid-stride
//   C  warp per 16 KiB (4 atoms of one block), grid-interleaved
// with a range of warps/SM; and the contiguous torch-like grid-stride copy.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mbshape scripts/microbench_shape.cu
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ int4 ld4(const char* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void st4(char* p, int4 v) {
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// A / C: warp copies CH bytes (CH = 4096 * NA) per unit; unit u = block u/(64K/CH), piece u%(...)
template <int NA>
__global__ void warp_units(const char* src, char* dst, const int32_t* ps, const int32_t* pd, long nunits) {
    constexpr int PER = 16 / NA;          // units per 64 KiB block
    const int lane = threadIdx.x & 31;
    const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
    for (long R = 0; R < nunits; R += 32 * nw) {
        const long mine = R + warp + (long)lane * nw;
        const char* s = nullptr;
        char* d = nullptr;
        if (mine < nunits) {
            s = src + (long)__ldg(ps + mine / PER) * 65536 + (mine % PER) * 4096 * NA;
            d = dst + (long)__ldg(pd + mine / PER) * 65536 + (mine % PER) * 4096 * NA;
        }
        for (int k = 0; k < 32; ++k) {
            const char* sk = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(s), k));
            char* dk = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(d), k));
            if (!sk) break;
            int4 v[8 * NA];
#pragma unroll
            for (int i = 0; i < 8 * NA; ++i) v[i] = ld4(sk + (i * 32 + lane) * 16);
#pragma unroll
            for (int i = 0; i < 8 * NA; ++i) st4(dk + (i * 32 + lane) * 16, v[i]);
        }
    }
}

// B: CTA per 64 KiB block
template <int T>
__global__ void __launch_bounds__(T) cta_blocks(const char* src, char* dst, const int32_t* ps, const int32_t* pd, long nblk) {
    constexpr int V = 65536 / 16 / T;   // 16-byte vectors per thread per block
    for (long b = blockIdx.x; b < nblk; b += gridDim.x) {
        const char* s = src + (long)__ldg(ps + b) * 65536;
        char* d = dst + (long)__ldg(pd + b) * 65536;
        int4 v[V];
#pragma unroll
        for (int i = 0; i < V; ++i) v[i] = ld4(s + (i * T + threadIdx.x) * 16);
#pragma unroll
        for (int i = 0; i < V; ++i) st4(d + (i * T + threadIdx.x) * 16, v[i]);
    }
}

__global__ void contig(const int4* __restrict__ a, int4* __restrict__ b, long n) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
    cudaSetDevice(0);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long foot = 80L << 30, moved = 16L << 30, nblk = moved / 65536, fblk = foot / 65536;
    char *a, *b;
    if (cudaMalloc(&a, foot) != cudaSuccess || cudaMalloc(&b, foot) != cudaSuccess) { printf("alloc failed\n"); return 1; }
    cudaMemset(a, 1, foot);
    cudaMemset(b, 2, foot);
    std::vector<int32_t> all(fblk), ps(nblk), pd(nblk);
    std::iota(all.begin(), all.end(), 0);
    std::mt19937 rng(3);
    std::shuffle(all.begin(), all.end(), rng);
    std::copy(all.begin(), all.begin() + nblk, ps.begin());
    std::shuffle(all.begin(), all.end(), rng);
    std::copy(all.begin(), all.begin() + nblk, pd.begin());
    int32_t *dps, *dpd;
    cudaMalloc(&dps, nblk * 4);
    cudaMalloc(&dpd, nblk * 4);
    cudaMemcpy(dps, ps.data(), nblk * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dpd, pd.data(), nblk * 4, cudaMemcpyHostToDevice);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](auto fn, const char* name) {
        for (int i = 0; i < 2; ++i) fn();
        float best = 1e9;
        for (int i = 0; i < 6; ++i) {
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        printf("%-48s %8.3f ms %7.1f GB/s\n", name, best, 2.0 * moved / best / 1e6);
    };
    char nm[96];
    for (int warps : {4, 6, 8, 12, 16}) {
        snprintf(nm, sizeof nm, "A warp/4KiB atom, %d warps/SM", warps);
        time([&] { warp_units<1><<<sms, 32 * warps>>>(a, b, dps, dpd, nblk * 16); }, nm);
    }
    for (int warps : {2, 4, 6, 8}) {
        snprintf(nm, sizeof nm, "C warp/16KiB, %d warps/SM", warps);
        time([&] { warp_units<4><<<sms, 32 * warps>>>(a, b, dps, dpd, nblk * 4); }, nm);
    }
    for (int per : {1, 2, 3, 4, 6, 8}) {
        snprintf(nm, sizeof nm, "B CTA(256)/64KiB block, %d CTAs/SM", per);
        time([&] { cta_blocks<256><<<sms * per, 256>>>(a, b, dps, dpd, nblk); }, nm);
    }
    for (int per : {1, 2, 4}) {
        snprintf(nm, sizeof nm, "B CTA(512)/64KiB block, %d CTAs/SM", per);
        time([&] { cta_blocks<512><<<sms * per, 512>>>(a, b, dps, dpd, nblk); }, nm);
    }
    for (int per : {4, 8, 16}) {
        snprintf(nm, sizeof nm, "contiguous grid-stride 256 thr, %d CTAs/SM", per);
        time([&] { contig<<<sms * per, 256>>>(reinterpret_cast<const int4*>(a), reinterpret_cast<int4*>(b), moved / 16); }, nm);
    }
    time([&] { cudaMemcpyAsync(b, a, moved, cudaMemcpyDeviceToDevice); }, "cudaMemcpy D2D contiguous");
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
