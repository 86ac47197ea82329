// microbench.cu -- what does the reshard kernel's structure reach on B200?
// Copies N 4-KiB atoms with the same warp-per-atom LDG/STG structure as
// flykv_reshard_kernel, for (a) contiguous, (b) source permuted in 64 KiB
// blocks, (c) both permuted, next to cudaMemcpy D2D of the same bytes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

__device__ __forceinline__ int4 ldn(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void stn(int4* p, int4 v) {
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// src atom a at src_blk[a / 16] * 16 + a % 16 (blocks of 16 atoms = 64 KiB)
template <int U>
__global__ void __launch_bounds__(256) copy_atoms(const char* src, char* dst, const int* sblk, const int* dblk, long n) {
    const int lane = threadIdx.x & 31;
    long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    long nw = ((long)gridDim.x * blockDim.x) >> 5;
    for (long a0 = warp * U; a0 < n; a0 += nw * U) {
        int4 v[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long a = a0 + u < n ? a0 + u : a0;
            const int4* s = reinterpret_cast<const int4*>(src + ((long)sblk[a >> 4] * 16 + (a & 15)) * 4096) + lane;
#pragma unroll
            for (int i = 0; i < 8; ++i) v[u][i] = ldn(s + i * 32);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long a = a0 + u;
            if (a >= n) break;
            int4* d = reinterpret_cast<int4*>(dst + ((long)dblk[a >> 4] * 16 + (a & 15)) * 4096) + lane;
#pragma unroll
            for (int i = 0; i < 8; ++i) stn(d + i * 32, v[u][i]);
        }
    }
}

int main(int argc, char** argv) {
    const long bytes = 19685965824L;
    const long n = bytes / 4096, nblk = n / 16;
    char *a, *b;
    int *ident, *perm1, *perm2;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    std::vector<int> h(nblk);
    for (long i = 0; i < nblk; ++i) h[i] = (int)i;
    cudaMalloc(&ident, nblk * 4);
    cudaMemcpy(ident, h.data(), nblk * 4, cudaMemcpyHostToDevice);
    std::mt19937 rng(1);
    std::shuffle(h.begin(), h.end(), rng);
    cudaMalloc(&perm1, nblk * 4);
    cudaMemcpy(perm1, h.data(), nblk * 4, cudaMemcpyHostToDevice);
    std::shuffle(h.begin(), h.end(), rng);
    cudaMalloc(&perm2, nblk * 4);
    cudaMemcpy(perm2, h.data(), nblk * 4, cudaMemcpyHostToDevice);
    cudaMemset(a, 1, bytes);
    cudaMemset(b, 2, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](auto fn, const char* name) {
        for (int i = 0; i < 3; ++i) fn();
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int i = 0; i < 10; ++i) {
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = std::min(best, ms);
        }
        printf("%-40s %8.3f ms  %7.1f GB/s (read+write)\n", name, best, 2.0 * bytes / best / 1e6);
    };
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    time([&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); }, "cudaMemcpy D2D");
    for (int per : {2, 4}) {
        int g = sms * per;
        char name[64];
        snprintf(name, 64, "contiguous U1 grid %d", g);
        time([&] { copy_atoms<1><<<g, 256>>>(a, b, ident, ident, n); }, name);
        snprintf(name, 64, "contiguous U2 grid %d", g);
        time([&] { copy_atoms<2><<<g, 256>>>(a, b, ident, ident, n); }, name);
        snprintf(name, 64, "src-permuted 64K U2 grid %d", g);
        time([&] { copy_atoms<2><<<g, 256>>>(a, b, perm1, ident, n); }, name);
        snprintf(name, 64, "both-permuted 64K U2 grid %d", g);
        time([&] { copy_atoms<2><<<g, 256>>>(a, b, perm1, perm2, n); }, name);
    }
    int g = sms * 16;
    time([&] { copy_atoms<1><<<g, 256>>>(a, b, ident, ident, n); }, "contiguous U1 grid 16/SM (non-persistent-ish)");
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
