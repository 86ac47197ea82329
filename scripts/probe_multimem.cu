// probe_multimem.cu -- NVLS multicast on this box's B200 (N2 rest).
//
// One GPU is visible, so the multicast object has one member: this checks
// that the driver path (cuMulticastCreate / AddDevice / BindMem / Map) and
// the sm_100a `multimem.st` instruction work, that a multimem store lands in
// the bound pool memory, and what one GPU's SMs can push through a multicast
// mapping against plain stores.  Fan-out to several GPUs needs more GPUs.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probe_multimem scripts/probe_multimem.cu -lcuda
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
    printf("FAIL %s: %s\n", #x, s_); return 1; } } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(r_)); \
    return 1; } } while (0)

__global__ void copy_uc(const int4* __restrict__ src, int4* dst, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
        asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(dst + i), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                     : "memory");
    }
}

// the same copy, stored through the multicast mapping: every member's bound
// memory receives the 16 bytes
__global__ void copy_mc(const int4* __restrict__ src, int4* mc, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int4 v;
        asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(src + i));
        asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i), "r"(v.x), "r"(v.y), "r"(v.z),
                     "r"(v.w)
                     : "memory");
    }
}

__global__ void fill(int4* p, int64_t n, int seed) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t h = (uint32_t)(i * 2654435761u) ^ (uint32_t)seed;
        p[i] = make_int4((int)h, (int)(h * 3u), (int)(h ^ 0x5bd1e995u), (int)(i & 0x7fffffff));
    }
}

int main() {
    RK(cudaSetDevice(0));
    RK(cudaFree(0));
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    int mcs = 0;
    CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("multicast_supported=%d\n", mcs);
    if (!mcs) return 0;
    size_t bytes = (size_t)4 << 30;  // 4 GiB: far larger than L2
    CUmulticastObjectProp mp;
    CUmemGenericAllocationHandle mc;
    size_t mgran = 0;
    bool made = false;
    const struct { CUmemAllocationHandleType t; const char* name; } kinds[] = {
        {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, "posix_fd"}, {CU_MEM_HANDLE_TYPE_FABRIC, "fabric"},
        {CU_MEM_HANDLE_TYPE_NONE, "none"}};
    for (const auto& k : kinds) {
        std::memset(&mp, 0, sizeof(mp));
        mp.numDevices = 1;
        mp.size = bytes;
        mp.handleTypes = k.t;
        CUresult g = cuMulticastGetGranularity(&mgran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
        if (g == CUDA_SUCCESS && mgran) mp.size = (bytes + mgran - 1) / mgran * mgran;
        CUresult r = cuMulticastCreate(&mc, &mp);
        const char* es = "";
        cuGetErrorString(r, &es);
        printf("cuMulticastCreate(numDevices=1, handle=%s, size=%zu, gran=%zu rc=%d): %d %s\n", k.name, mp.size, mgran,
               (int)g, (int)r, es);
        if (r == CUDA_SUCCESS) { made = true; break; }
    }
    if (!made) return 1;
    bytes = mp.size;
    CK(cuMulticastAddDevice(mc, dev));
    CUmemAllocationProp ap;
    std::memset(&ap, 0, sizeof(ap));
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    size_t agran = 0;
    CK(cuMemGetAllocationGranularity(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    printf("granularity: multicast %zu, allocation %zu, size %zu\n", mgran, agran, bytes);
    CUmemGenericAllocationHandle mem;
    CK(cuMemCreate(&mem, bytes, &ap, 0));
    CK(cuMulticastBindMem(mc, 0, mem, 0, bytes, 0));
    CUmemAccessDesc acc;
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = 0;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUdeviceptr uc = 0, mva = 0;
    CK(cuMemAddressReserve(&uc, bytes, mgran, 0, 0));
    CK(cuMemMap(uc, bytes, 0, mem, 0));
    CK(cuMemSetAccess(uc, bytes, &acc, 1));
    CK(cuMemAddressReserve(&mva, bytes, mgran, 0, 0));
    CK(cuMemMap(mva, bytes, 0, mc, 0));
    CK(cuMemSetAccess(mva, bytes, &acc, 1));

    int4* src = nullptr;
    RK(cudaMalloc(&src, bytes));
    const int64_t n = (int64_t)(bytes / 16);
    int sms = 0;
    RK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    fill<<<sms * 8, 256>>>(src, n, 7);
    RK(cudaMemset(reinterpret_cast<void*>(uc), 0, bytes));
    RK(cudaDeviceSynchronize());

    // correctness: a multimem store lands in the bound memory (read back through the unicast mapping)
    copy_mc<<<sms * 8, 256>>>(src, reinterpret_cast<int4*>(mva), n);
    RK(cudaGetLastError());
    RK(cudaDeviceSynchronize());
    std::vector<int4> a(1 << 20), b(1 << 20);
    size_t bad = 0;
    for (size_t off : {(size_t)0, bytes / 2, bytes - a.size() * 16}) {
        RK(cudaMemcpy(a.data(), reinterpret_cast<char*>(src) + off, a.size() * 16, cudaMemcpyDeviceToHost));
        RK(cudaMemcpy(b.data(), reinterpret_cast<void*>(uc + off), b.size() * 16, cudaMemcpyDeviceToHost));
        bad += std::memcmp(a.data(), b.data(), a.size() * 16) != 0;
    }
    printf("multimem.st -> bound memory: %s\n", bad ? "MISMATCH" : "bytes match (3 x 16 MiB windows)");

    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int shape : {4, 8, 16}) {
        for (int which = 0; which < 2; ++which) {
            float best = 1e30f;
            for (int rep = 0; rep < 5; ++rep) {
                cudaEventRecord(e0);
                if (which == 0) copy_uc<<<sms * shape, 256>>>(src, reinterpret_cast<int4*>(uc), n);
                else copy_mc<<<sms * shape, 256>>>(src, reinterpret_cast<int4*>(mva), n);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            printf("%s copy, %d CTAs/SM x 256: %.3f ms, %.1f GB/s (read + write)\n",
                   which ? "multimem" : "unicast", shape, best, 2.0 * bytes / best / 1e6);
        }
    }
    RK(cudaGetLastError());
    return bad ? 1 : 0;
}
