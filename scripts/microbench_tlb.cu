// microbench_tlb.cu -- is the re-layout's gap to a contiguous copy a TLB
// effect?  Copy 4 KiB atoms, 16 per 64 KiB block, blocks in a seeded random
// permutation (source and destination independently), warp per atom,
// grid-interleaved (the reshard's structure, no decode), over footprints from
// 2 GiB to 96 GiB per side, in memory from cudaMalloc and from one cuMemCreate
// allocation mapped with 2 MiB or 512 MiB VA alignment; next to the same
// copy with contiguous blocks.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/mbtlb scripts/microbench_tlb.cu -lcuda
#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <random>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ int4 ld4(const char* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}
__device__ __forceinline__ void st4(char* p, int4 v) {
    asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// The reshard's structure without its decode: grid-interleaved slots (step
// k of round R of warp w is atom R + k*nwarps + w), lane-parallel address
// fetch one round ahead (lane k fetches step k's block index), two atoms in
// flight per warp; atom a = block a/16 of the permutation, atom a%16 in it.
__global__ void __launch_bounds__(192) copy_perm(const char* src, char* dst, const int32_t* ps, const int32_t* pd, long natoms) {
    const int lane = threadIdx.x & 31;
    const long warp = ((long)blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = ((long)gridDim.x * blockDim.x) >> 5;
    auto fetch = [&](long R, const char*& s, char*& d) {
        const long a = R + warp + (long)lane * nw;
        s = nullptr;
        d = nullptr;
        if (a < natoms) {
            s = src + (long)__ldg(ps + (a >> 4)) * 65536 + (a & 15) * 4096;
            d = dst + (long)__ldg(pd + (a >> 4)) * 65536 + (a & 15) * 4096;
        }
    };
    const char* s;
    char* d;
    fetch(0, s, d);
    for (long R = 0; R < natoms; R += 32 * nw) {
        const char* sn;
        char* dn;
        bool fetched = false;
        for (int k0 = 0; k0 < 32; k0 += 2) {
            int4 v[2][8];
            const char* ss[2];
            char* dd[2];
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                ss[u] = reinterpret_cast<const char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(s), k0 + u));
                dd[u] = reinterpret_cast<char*>(__shfl_sync(0xffffffffu, reinterpret_cast<uintptr_t>(d), k0 + u));
                if (ss[u])
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[u][i] = ld4(ss[u] + (i * 32 + lane) * 16);
            }
            if (!fetched) {
                fetch(R + 32 * nw, sn, dn);
                fetched = true;
            }
#pragma unroll
            for (int u = 0; u < 2; ++u)
                if (dd[u])
#pragma unroll
                    for (int i = 0; i < 8; ++i) st4(dd[u] + (i * 32 + lane) * 16, v[u][i]);
        }
        s = sn;
        d = dn;
    }
}

int main() {
    cuInit(0);
    cudaSetDevice(0);
    cudaFree(0);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long moved = 16L << 30;                 // bytes copied per launch
    const long nblk_moved = moved / 65536;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](const char* tag, char* a, char* b, long foot) {
        const long nblk = foot / 65536;
        for (int mode = 0; mode < 2; ++mode) {   // 0 contiguous, 1 random permutation
            std::vector<int32_t> ps(nblk_moved), pd(nblk_moved);
            std::vector<int32_t> all(nblk);
            std::iota(all.begin(), all.end(), 0);
            std::mt19937 rng(7);
            if (mode) std::shuffle(all.begin(), all.end(), rng);
            for (long i = 0; i < nblk_moved; ++i) ps[i] = all[i % nblk];
            if (mode) std::shuffle(all.begin(), all.end(), rng);
            for (long i = 0; i < nblk_moved; ++i) pd[i] = all[i % nblk];
            int32_t *dps, *dpd;
            cudaMalloc(&dps, nblk_moved * 4);
            cudaMalloc(&dpd, nblk_moved * 4);
            cudaMemcpy(dps, ps.data(), nblk_moved * 4, cudaMemcpyHostToDevice);
            cudaMemcpy(dpd, pd.data(), nblk_moved * 4, cudaMemcpyHostToDevice);
            float best = 1e9;
            for (int r = 0; r < 8; ++r) {
                cudaEventRecord(e0);
                copy_perm<<<sms, 192>>>(a, b, dps, dpd, nblk_moved * 16);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (r >= 2) best = std::min(best, ms);
            }
            printf("%-28s footprint %6.1f GiB per side %-11s %8.3f ms %7.1f GB/s\n", tag, foot / 1073741824.0,
                   mode ? "permuted" : "contiguous", best, 2.0 * moved / best / 1e6);
            cudaFree(dps);
            cudaFree(dpd);
        }
    };
    const long maxfoot = 80L << 30;
    {
        char *a, *b;
        if (cudaMalloc(&a, maxfoot) != cudaSuccess || cudaMalloc(&b, maxfoot) != cudaSuccess) { printf("alloc failed\n"); return 1; }
        cudaMemset(a, 1, maxfoot);
        cudaMemset(b, 2, maxfoot);
        for (long f : {16L << 30, 32L << 30, 80L << 30}) run("cudaMalloc", a, b, f);
        cudaFree(a);
        cudaFree(b);
    }
    for (size_t align : {(size_t)2 << 20, (size_t)512 << 20}) {
        CUmemAllocationProp prop;
        memset(&prop, 0, sizeof prop);
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop.location.id = 0;
        CUdeviceptr va[2];
        CUmemGenericAllocationHandle h[2];
        bool ok = true;
        for (int k = 0; k < 2; ++k) {
            ok = ok && cuMemCreate(&h[k], maxfoot, &prop, 0) == CUDA_SUCCESS;
            ok = ok && cuMemAddressReserve(&va[k], maxfoot, align, 0, 0) == CUDA_SUCCESS;
            ok = ok && cuMemMap(va[k], maxfoot, 0, h[k], 0) == CUDA_SUCCESS;
            CUmemAccessDesc acc;
            acc.location = prop.location;
            acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
            ok = ok && cuMemSetAccess(va[k], maxfoot, &acc, 1) == CUDA_SUCCESS;
        }
        if (!ok) { printf("VMM alloc failed (align %zu)\n", align); continue; }
        cudaMemset((void*)va[0], 1, maxfoot);
        cudaMemset((void*)va[1], 2, maxfoot);
        char tag[64];
        snprintf(tag, sizeof tag, "cuMemCreate align %zu MiB", align >> 20);
        for (long f : {16L << 30, 80L << 30}) run(tag, (char*)va[0], (char*)va[1], f);
        for (int k = 0; k < 2; ++k) {
            cuMemUnmap(va[k], maxfoot);
            cuMemAddressFree(va[k], maxfoot);
            cuMemRelease(h[k]);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
