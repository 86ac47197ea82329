// microbench_v8.cu -- 128-bit vs 256-bit (sm_100 LDG/STG.256) global accesses
// for the reshard's warp-per-4KiB-atom copy, write-only and with R-fold
// replication (GQA, R = p/H), next to cudaMemset / cudaMemcpy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbv8 microbench_v8.cu
#include <algorithm>
#include <cstdio>
#include <cuda_runtime.h>

struct V4 { int x[4]; };
struct V8 { int x[8]; };

__device__ __forceinline__ void ld(V4& r, const char* p) {
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x[0]), "=r"(r.x[1]), "=r"(r.x[2]), "=r"(r.x[3]) : "l"(p));
}
__device__ __forceinline__ void st(char* p, const V4& v) {
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x[0]), "r"(v.x[1]), "r"(v.x[2]), "r"(v.x[3]) : "memory");
}
__device__ __forceinline__ void ld(V8& r, const char* p) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r.x[0]), "=r"(r.x[1]), "=r"(r.x[2]), "=r"(r.x[3]), "=r"(r.x[4]), "=r"(r.x[5]), "=r"(r.x[6]), "=r"(r.x[7]) : "l"(p));
}
__device__ __forceinline__ void st(char* p, const V8& v) {
    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.x[0]), "r"(v.x[1]), "r"(v.x[2]),
                 "r"(v.x[3]), "r"(v.x[4]), "r"(v.x[5]), "r"(v.x[6]), "r"(v.x[7]) : "memory");
}

// atom a of n_src -> dst region r < R at position a.  U atoms per warp in flight.
template <class V, int U>
__global__ void __launch_bounds__(512) rep(const char* src, char* dst, long n_src, int R, int write_only) {
    constexpr int VB = sizeof(V), NI = 4096 / (32 * VB);
    const int lane = threadIdx.x & 31;
    long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    long nw = ((long)gridDim.x * blockDim.x) >> 5;
    for (long a0 = warp * U; a0 < n_src; a0 += nw * U) {
        V v[U][NI];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            long a = min(a0 + u, n_src - 1);
#pragma unroll
            for (int i = 0; i < NI; ++i) {
                if (write_only) {
#pragma unroll
                    for (int k = 0; k < VB / 4; ++k) v[u][i].x[k] = (int)a + i + k;
                } else {
                    ld(v[u][i], src + a * 4096 + (i * 32 + lane) * VB);
                }
            }
        }
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                long a = a0 + u;
                if (a >= n_src) break;
#pragma unroll
                for (int i = 0; i < NI; ++i) st(dst + ((long)r * n_src + a) * 4096 + (i * 32 + lane) * VB, v[u][i]);
            }
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
        printf("%-48s best %8.3f ms %7.1f GB/s  mean %7.1f GB/s\n", name, best, traffic / best / 1e6, traffic / (sum / 10) / 1e6);
    };
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    time([&] { cudaMemsetAsync(b, 3, bytes); }, "cudaMemset (write only)", (double)bytes);
    time([&] { cudaMemcpyAsync(b, a, bytes, cudaMemcpyDeviceToDevice); }, "cudaMemcpy D2D", 2.0 * bytes);
    char name[128];
    for (int wo = 1; wo >= 0; --wo) {
        for (int R : {1, 2, 8}) {
            if (wo && R > 1) continue;
            long n_src = bytes / 4096 / R;
            double traffic = wo ? (double)bytes : (double)bytes * (1.0 + 1.0 / R);
            for (int warps : {6, 8, 10, 12, 16}) {
                snprintf(name, 128, "%s R=%d v4 U2 %d warps/SM", wo ? "write-only" : "copy", R, warps);
                time([&] { rep<V4, 2><<<sms, 32 * warps>>>(a, b, n_src, R, wo); }, name, traffic);
                snprintf(name, 128, "%s R=%d v8 U2 %d warps/SM", wo ? "write-only" : "copy", R, warps);
                time([&] { rep<V8, 2><<<sms, 32 * warps>>>(a, b, n_src, R, wo); }, name, traffic);
                snprintf(name, 128, "%s R=%d v8 U1 %d warps/SM", wo ? "write-only" : "copy", R, warps);
                time([&] { rep<V8, 1><<<sms, 32 * warps>>>(a, b, n_src, R, wo); }, name, traffic);
            }
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
