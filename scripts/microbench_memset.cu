// microbench_memset.cu -- is cudaMemset's 7.4 TB/s an SM store rate or a
// data-dependent effect?  Grid-stride 16 B stores of a constant vs of
// varying data, next to cudaMemset of the same 16 GiB.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mbms microbench_memset.cu
#include <algorithm>
#include <cstdio>
#include <cuda_runtime.h>

template <int CONST>
__global__ void w(char* dst, long n16) {
    long t = (long)blockIdx.x * blockDim.x + threadIdx.x, nt = (long)gridDim.x * blockDim.x;
    for (long i = t; i < n16; i += nt) {
        int4 v = CONST ? make_int4(0x03030303, 0x03030303, 0x03030303, 0x03030303)
                       : make_int4((int)i, (int)(i * 3), (int)(i * 7), (int)(i * 11));
        asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(dst + i * 16), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
    }
}

int main() {
    const long bytes = 16L << 30;
    char* b;
    cudaMalloc(&b, bytes);
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
        printf("%-44s best %8.3f ms %7.1f GB/s\n", name, best, bytes / best / 1e6);
    };
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    time([&] { cudaMemsetAsync(b, 3, bytes); }, "cudaMemset 0x03");
    time([&] { cudaMemsetAsync(b, 0, bytes); }, "cudaMemset 0x00");
    time([&] { w<1><<<sms * 4, 256>>>(b, bytes / 16); }, "kernel, constant 0x03 data");
    time([&] { w<0><<<sms * 4, 256>>>(b, bytes / 16); }, "kernel, varying data");
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
