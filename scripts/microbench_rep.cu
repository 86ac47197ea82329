// microbench_rep.cu -- ceiling of the GQA-replicating re-layout on B200.
// Reads n/R 4-KiB atoms and writes each to R destination regions (the
// write-heavy traffic of TP > kv_heads, R = p/H), with the reshard kernel's
// warp-per-atom LDG/STG structure, next to cudaMemset (write-only) and
// cudaMemcpy D2D of the same destination bytes.  Reports read+write GB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbr microbench_rep.cu
#include <algorithm>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int4 ldn(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void stn(int4* p, int4 v) {
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// source atom a (n_src of them) -> dst region r (r < R), position a
__global__ void __launch_bounds__(320) rep_atoms(const char* src, char* dst, long n_src, int R) {
    const int lane = threadIdx.x & 31;
    long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    long nw = ((long)gridDim.x * blockDim.x) >> 5;
    for (long a = warp; a < n_src; a += nw) {
        int4 v[8];
        const int4* s = reinterpret_cast<const int4*>(src + a * 4096) + lane;
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = ldn(s + i * 32);
        for (int r = 0; r < R; ++r) {
            int4* d = reinterpret_cast<int4*>(dst + ((long)r * n_src + a) * 4096) + lane;
#pragma unroll
            for (int i = 0; i < 8; ++i) stn(d + i * 32, v[i]);
        }
    }
}

int main() {
    const long bytes = 16L << 30;  // destination bytes
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
        printf("%-44s best %8.3f ms %7.1f GB/s  mean %7.1f GB/s\n", name, best, traffic / best / 1e6, traffic / (sum / 10) / 1e6);
    };
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    time([&] { cudaMemsetAsync(b, 3, bytes); }, "cudaMemset (write only)", (double)bytes);
    time([&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); }, "cudaMemcpy D2D", 2.0 * bytes);
    for (int R : {1, 2, 4, 8}) {
        long n_src = bytes / 4096 / R;
        for (int thr : {192, 256, 320}) {
            char name[96];
            snprintf(name, 96, "replicate R=%d, %d thr x 1 CTA/SM", R, thr);
            time([&] { rep_atoms<<<sms, thr>>>(a, b, n_src, R); }, name, (double)bytes * (1.0 + 1.0 / R));
            snprintf(name, 96, "replicate R=%d, %d thr x 2 CTA/SM", R, thr);
            time([&] { rep_atoms<<<2 * sms, thr>>>(a, b, n_src, R); }, name, (double)bytes * (1.0 + 1.0 / R));
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
