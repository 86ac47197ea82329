// flykv_vmm.cpp -- the Model Weights Manager's contiguous zero-copy view
// (Eq.1): "the active weights used for TP execution are contiguous
// in virtual memory but map to the existing physical memory of the DP
// replica".  Weights allocated through kv_vmm_alloc (cuMemCreate) can have a
// rank's row segments (Q, K, V slices of the fused W^QKV, or the rows of a
// column-parallel matrix) mapped back to back into a fresh virtual range that
// aliases the same physical memory: one contiguous [rows, cols] operand for
// the GEMM, 0 bytes copied.  cuMemMap only maps whole physical allocations
// (offset 0), so a weight buffer is built from granularity-sized physical
// chunks mapped back to back; an alias maps the chunks its segments cover.
//
// Driver-API entry points are resolved at run time with
// cudaGetDriverEntryPoint, so libflykv.so does not link libcuda.
#include <cuda.h>

#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "flykv.h"
#include "flykv_internal.h"

extern kv_status flykv_fail(kv_status s, const char* fmt, ...);

namespace {

struct Drv {
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
    bool ok = false;
};

template <typename F>
bool resolve(const char* name, F& fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || !p ||
        q != cudaDriverEntryPointSuccess)
        return false;
    fn = reinterpret_cast<F>(p);
    return true;
}

Drv& drv() {
    static Drv d;
    static std::once_flag once;
    std::call_once(once, [] {
        d.ok = resolve("cuMemCreate", d.create) && resolve("cuMemRelease", d.release) &&
               resolve("cuMemAddressReserve", d.reserve) && resolve("cuMemAddressFree", d.addr_free) &&
               resolve("cuMemMap", d.map) && resolve("cuMemUnmap", d.unmap) &&
               resolve("cuMemSetAccess", d.set_access) &&
               resolve("cuMemGetAllocationGranularity", d.granularity);
    });
    return d;
}

CUmemAllocationProp prop_for(int device) {
    CUmemAllocationProp prop;
    std::memset(&prop, 0, sizeof prop);
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    return prop;
}

}  // namespace

struct kv_vmm_buffer {
    int device;
    size_t chunk;                                    // physical chunk bytes (= granularity)
    std::vector<CUmemGenericAllocationHandle> handles;
    CUdeviceptr va;
    size_t bytes;
};

#define DRV_TRY(call, what)                                                       \
    do {                                                                          \
        CUresult _r = (call);                                                     \
        if (_r != CUDA_SUCCESS) return flykv_fail(KV_ERR_CUDA, "%s failed (%d)", what, (int)_r); \
    } while (0)

extern "C" kv_status kv_vmm_granularity(int32_t device, uint64_t* gran) {
    if (!gran) return flykv_fail(KV_ERR_INVALID_ARG, "gran is NULL");
    Drv& d = drv();
    if (!d.ok) return flykv_fail(KV_ERR_CUDA, "CUDA VMM driver entry points unavailable");
    CUmemAllocationProp prop = prop_for(device);
    size_t g = 0;
    DRV_TRY(d.granularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "cuMemGetAllocationGranularity");
    *gran = g;
    return KV_OK;
}

static void release_buffer(Drv& d, kv_vmm_buffer* b, size_t mapped) {
    if (mapped) d.unmap(b->va, mapped);
    if (b->va) d.addr_free(b->va, b->bytes);
    for (CUmemGenericAllocationHandle h : b->handles) d.release(h);
    delete b;
}

extern "C" kv_status kv_vmm_alloc(int32_t device, uint64_t bytes, kv_vmm_buffer** out, void** dptr) {
    if (!out || !dptr || bytes == 0) return flykv_fail(KV_ERR_INVALID_ARG, "bad kv_vmm_alloc arguments");
    Drv& d = drv();
    if (!d.ok) return flykv_fail(KV_ERR_CUDA, "CUDA VMM driver entry points unavailable");
    uint64_t g = 0;
    kv_status s = kv_vmm_granularity(device, &g);
    if (s) return s;
    const size_t size = (bytes + g - 1) / g * g;
    CUmemAllocationProp prop = prop_for(device);
    kv_vmm_buffer* b = new (std::nothrow) kv_vmm_buffer();
    if (!b) return flykv_fail(KV_ERR_INVALID_ARG, "out of host memory");
    b->device = device;
    b->chunk = g;
    b->bytes = size;
    b->va = 0;
    CUresult r = d.reserve(&b->va, size, g, 0, 0);
    if (r != CUDA_SUCCESS) {
        b->va = 0;
        release_buffer(d, b, 0);
        return flykv_fail(KV_ERR_CUDA, "cuMemAddressReserve(%zu) failed (%d)", size, (int)r);
    }
    size_t mapped = 0;
    for (size_t off = 0; off < size; off += g) {
        CUmemGenericAllocationHandle h;
        r = d.create(&h, g, &prop, 0);
        if (r != CUDA_SUCCESS) break;
        b->handles.push_back(h);
        r = d.map(b->va + off, g, 0, h, 0);
        if (r != CUDA_SUCCESS) break;
        mapped += g;
    }
    if (r == CUDA_SUCCESS) {
        CUmemAccessDesc acc;
        acc.location = prop.location;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        r = d.set_access(b->va, size, &acc, 1);
    }
    if (r != CUDA_SUCCESS) {
        release_buffer(d, b, mapped);
        return flykv_fail(KV_ERR_CUDA, "VMM allocation of the weight buffer failed (%d)", (int)r);
    }
    *out = b;
    *dptr = reinterpret_cast<void*>(b->va);
    return KV_OK;
}

extern "C" kv_status kv_vmm_free(kv_vmm_buffer* b) {
    if (!b) return KV_OK;
    Drv& d = drv();
    release_buffer(d, b, b->bytes);
    return KV_OK;
}

extern "C" kv_status weight_view_alias(const kv_vmm_buffer* b, const kv_view* v, void** contiguous, uint64_t* bytes) {
    if (!b || !v || !contiguous || !bytes || v->n_seg < 1 || v->n_seg > 3)
        return flykv_fail(KV_ERR_INVALID_ARG, "bad weight_view_alias arguments");
    Drv& d = drv();
    if (!d.ok) return flykv_fail(KV_ERR_CUDA, "CUDA VMM driver entry points unavailable");
    uint64_t g = 0;
    kv_status s = kv_vmm_granularity(b->device, &g);
    if (s) return s;
    size_t offs[3], lens[3], total = 0;
    for (int k = 0; k < v->n_seg; ++k) {
        const kv_view_segment& sg = v->seg[k];
        if (sg.ld != sg.cols)
            return flykv_fail(KV_ERR_INVALID_ARG, "segment %d is strided (row-parallel view): not a row range", k);
        const uintptr_t p = reinterpret_cast<uintptr_t>(sg.ptr);
        if (p < b->va || p >= b->va + b->bytes) return flykv_fail(KV_ERR_INVALID_ARG, "segment %d outside the buffer", k);
        offs[k] = p - b->va;
        lens[k] = (size_t)(sg.rows * sg.cols * v->elem_bytes);
        if (offs[k] % g || lens[k] % g || offs[k] + lens[k] > b->bytes)
            return flykv_fail(KV_ERR_INDIVISIBLE_EXTENT,
                              "segment %d (offset %zu, %zu bytes) not aligned to the %llu-byte VMM granularity", k,
                              offs[k], lens[k], (unsigned long long)g);
        total += lens[k];
    }
    CUdeviceptr va = 0;
    DRV_TRY(d.reserve(&va, total, g, 0, 0), "cuMemAddressReserve");
    size_t at = 0;
    for (int k = 0; k < v->n_seg; ++k) {
        for (size_t o = offs[k]; o < offs[k] + lens[k]; o += b->chunk) {
            CUresult r = d.map(va + at, b->chunk, 0, b->handles[o / b->chunk], 0);
            if (r != CUDA_SUCCESS) {
                if (at) d.unmap(va, at);
                d.addr_free(va, total);
                return flykv_fail(KV_ERR_CUDA, "cuMemMap of segment %d failed (%d)", k, (int)r);
            }
            at += b->chunk;
        }
    }
    CUmemAccessDesc acc;
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = b->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CUresult r = d.set_access(va, total, &acc, 1);
    if (r != CUDA_SUCCESS) {
        d.unmap(va, total);
        d.addr_free(va, total);
        return flykv_fail(KV_ERR_CUDA, "cuMemSetAccess failed (%d)", (int)r);
    }
    *contiguous = reinterpret_cast<void*>(va);
    *bytes = total;
    return KV_OK;
}

extern "C" kv_status weight_view_unalias(void* contiguous, uint64_t bytes) {
    if (!contiguous) return KV_OK;
    Drv& d = drv();
    if (!d.ok) return flykv_fail(KV_ERR_CUDA, "CUDA VMM driver entry points unavailable");
    const CUdeviceptr va = reinterpret_cast<CUdeviceptr>(contiguous);
    DRV_TRY(d.unmap(va, bytes), "cuMemUnmap");
    DRV_TRY(d.addr_free(va, bytes), "cuMemAddressFree");
    return KV_OK;
}
