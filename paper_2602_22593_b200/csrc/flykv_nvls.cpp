// flykv_nvls.cpp -- shareable pool memory and NVLS multicast teams for GQA
// head replication (Eq.3 replication P:536-541).
//
// When the destination degree p exceeds the KV head count H, every head is
// held by p/H ranks, an aligned team of engines at the same block IDs (R2,
// R6) and the same offsets (H_loc = 1).  A multicast object bound to the
// pools of such a team lets a sender that is a member of the team write an
// atom once (multimem.st) and have NVSwitch deliver it to every replica, so
// its NVLink egress is one copy instead of p/H (weight views
// follow any head set, so the pools of a team can be bound together).
//
// Pool memory for this path is one physical allocation per pool (cuMemCreate,
// POSIX file-descriptor shareable) instead of a cudaMalloc'ed torch tensor:
// multicast objects bind physical allocations, and peers map the pool
// through the exported descriptor (kv_pool_export / kv_pool_import) instead
// of CUDA IPC.  Driver entry points are resolved at run time; nothing here
// runs unless the caller asks for it, and kv_mc_supported reports whether the
// driver accepts a multicast object of the team size at all.
#include <cuda.h>
#include <unistd.h>

#include <cstring>
#include <mutex>
#include <new>

#include "flykv.h"
#include "flykv_internal.h"

extern kv_status flykv_fail(kv_status s, const char* fmt, ...);

namespace {

struct NvlsDrv {
    decltype(&cuMemCreate) create = nullptr;
    decltype(&cuMemRelease) release = nullptr;
    decltype(&cuMemAddressReserve) reserve = nullptr;
    decltype(&cuMemAddressFree) addr_free = nullptr;
    decltype(&cuMemMap) map = nullptr;
    decltype(&cuMemUnmap) unmap = nullptr;
    decltype(&cuMemSetAccess) set_access = nullptr;
    decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
    decltype(&cuMemExportToShareableHandle) export_handle = nullptr;
    decltype(&cuMemImportFromShareableHandle) import_handle = nullptr;
    decltype(&cuMulticastCreate) mc_create = nullptr;
    decltype(&cuMulticastAddDevice) mc_add = nullptr;
    decltype(&cuMulticastBindMem) mc_bind = nullptr;
    decltype(&cuMulticastUnbind) mc_unbind = nullptr;
    decltype(&cuMulticastGetGranularity) mc_gran = nullptr;
    decltype(&cuDeviceGet) device_get = nullptr;
    decltype(&cuGetErrorString) err = nullptr;
    bool ok = false, mc_ok = false;
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

NvlsDrv& drv() {
    static NvlsDrv d;
    static std::once_flag once;
    std::call_once(once, [] {
        d.ok = resolve("cuMemCreate", d.create) && resolve("cuMemRelease", d.release) &&
               resolve("cuMemAddressReserve", d.reserve) && resolve("cuMemAddressFree", d.addr_free) &&
               resolve("cuMemMap", d.map) && resolve("cuMemUnmap", d.unmap) &&
               resolve("cuMemSetAccess", d.set_access) &&
               resolve("cuMemGetAllocationGranularity", d.granularity) &&
               resolve("cuMemExportToShareableHandle", d.export_handle) &&
               resolve("cuMemImportFromShareableHandle", d.import_handle) && resolve("cuDeviceGet", d.device_get) &&
               resolve("cuGetErrorString", d.err);
        d.mc_ok = d.ok && resolve("cuMulticastCreate", d.mc_create) && resolve("cuMulticastAddDevice", d.mc_add) &&
                  resolve("cuMulticastBindMem", d.mc_bind) && resolve("cuMulticastUnbind", d.mc_unbind) &&
                  resolve("cuMulticastGetGranularity", d.mc_gran);
    });
    return d;
}

const char* errstr(CUresult r) {
    const char* s = "unknown";
    if (drv().err) drv().err(r, &s);
    return s;
}

#define NV_TRY(call, what)                                                                               \
    do {                                                                                                 \
        CUresult _r = (call);                                                                            \
        if (_r != CUDA_SUCCESS) return flykv_fail(KV_ERR_CUDA, "%s failed (%d: %s)", what, (int)_r, errstr(_r)); \
    } while (0)

CUmemAllocationProp pool_prop(int device) {
    CUmemAllocationProp prop;
    std::memset(&prop, 0, sizeof prop);
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    return prop;
}

// Map `h` (bytes, a whole allocation) read-write for `device` at a fresh VA.
kv_status map_rw(NvlsDrv& d, CUmemGenericAllocationHandle h, size_t bytes, size_t align, int device, CUdeviceptr* va) {
    *va = 0;
    NV_TRY(d.reserve(va, bytes, align, 0, 0), "cuMemAddressReserve");
    CUresult r = d.map(*va, bytes, 0, h, 0);
    if (r == CUDA_SUCCESS) {
        CUmemAccessDesc acc;
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc.location.id = device;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        r = d.set_access(*va, bytes, &acc, 1);
        if (r != CUDA_SUCCESS) d.unmap(*va, bytes);
    }
    if (r != CUDA_SUCCESS) {
        d.addr_free(*va, bytes);
        *va = 0;
        return flykv_fail(KV_ERR_CUDA, "cuMemMap / cuMemSetAccess failed (%d: %s)", (int)r, errstr(r));
    }
    return KV_OK;
}

}  // namespace

struct kv_pool_mem {
    CUmemGenericAllocationHandle h;
    CUdeviceptr va;
    size_t bytes;
    int device;  // the device the mapping was made accessible to
};

struct kv_mc {
    CUmemGenericAllocationHandle h;
    size_t bytes;
    int32_t n_devices;
    CUdeviceptr va = 0;   // this process's multicast mapping (kv_mc_map)
    int bound_device = -1;
    size_t bound_bytes = 0;
};

extern "C" kv_status kv_pool_alloc(int32_t device, uint64_t bytes, uint64_t align, kv_pool_mem** out, void** dptr) {
    if (!out || !dptr || bytes == 0) return flykv_fail(KV_ERR_INVALID_ARG, "bad kv_pool_alloc arguments");
    NvlsDrv& d = drv();
    if (!d.ok) return flykv_fail(KV_ERR_CUDA, "CUDA VMM driver entry points unavailable");
    CUmemAllocationProp prop = pool_prop(device);
    size_t g = 0;
    NV_TRY(d.granularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
    if (align > g) {
        if (align % g) return flykv_fail(KV_ERR_INVALID_ARG, "align %llu is not a multiple of the %zu-byte granularity",
                                         (unsigned long long)align, g);
        g = (size_t)align;
    }
    const size_t size = (bytes + g - 1) / g * g;
    kv_pool_mem* p = new (std::nothrow) kv_pool_mem();
    if (!p) return flykv_fail(KV_ERR_INVALID_ARG, "out of host memory");
    CUresult r = d.create(&p->h, size, &prop, 0);
    if (r != CUDA_SUCCESS) {
        delete p;
        return flykv_fail(KV_ERR_CUDA, "cuMemCreate(%zu) failed (%d: %s)", size, (int)r, errstr(r));
    }
    kv_status s = map_rw(d, p->h, size, g, device, &p->va);
    if (s) {
        d.release(p->h);
        delete p;
        return s;
    }
    p->bytes = size;
    p->device = device;
    *out = p;
    *dptr = reinterpret_cast<void*>(p->va);
    return KV_OK;
}

extern "C" kv_status kv_pool_export(const kv_pool_mem* p, int32_t* fd) {
    if (!p || !fd) return flykv_fail(KV_ERR_INVALID_ARG, "bad kv_pool_export arguments");
    NvlsDrv& d = drv();
    int f = -1;
    NV_TRY(d.export_handle(&f, p->h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0), "cuMemExportToShareableHandle");
    *fd = f;
    return KV_OK;
}

extern "C" kv_status kv_pool_import(int32_t fd, uint64_t bytes, int32_t device, kv_pool_mem** out, void** dptr) {
    if (fd < 0 || !out || !dptr || bytes == 0) return flykv_fail(KV_ERR_INVALID_ARG, "bad kv_pool_import arguments");
    NvlsDrv& d = drv();
    if (!d.ok) return flykv_fail(KV_ERR_CUDA, "CUDA VMM driver entry points unavailable");
    kv_pool_mem* p = new (std::nothrow) kv_pool_mem();
    if (!p) return flykv_fail(KV_ERR_INVALID_ARG, "out of host memory");
    CUresult r = d.import_handle(&p->h, reinterpret_cast<void*>((uintptr_t)fd), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    if (r != CUDA_SUCCESS) {
        delete p;
        return flykv_fail(KV_ERR_CUDA, "cuMemImportFromShareableHandle failed (%d: %s)", (int)r, errstr(r));
    }
    CUmemAllocationProp prop = pool_prop(device);
    size_t g = 0;
    d.granularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    kv_status s = map_rw(d, p->h, bytes, g ? g : (2u << 20), device, &p->va);
    if (s) {
        d.release(p->h);
        delete p;
        return s;
    }
    p->bytes = bytes;
    p->device = device;
    *out = p;
    *dptr = reinterpret_cast<void*>(p->va);
    return KV_OK;
}

extern "C" kv_status kv_pool_free(kv_pool_mem* p) {
    if (!p) return KV_OK;
    NvlsDrv& d = drv();
    if (p->va) {
        d.unmap(p->va, p->bytes);
        d.addr_free(p->va, p->bytes);
    }
    d.release(p->h);
    delete p;
    return KV_OK;
}

extern "C" kv_status kv_mc_supported(int32_t n_devices, uint64_t bytes, int32_t* ok, uint64_t* granularity) {
    if (!ok || n_devices < 1 || bytes == 0) return flykv_fail(KV_ERR_INVALID_ARG, "bad kv_mc_supported arguments");
    *ok = 0;
    if (granularity) *granularity = 0;
    NvlsDrv& d = drv();
    if (!d.mc_ok) return flykv_fail(KV_ERR_CUDA, "multicast driver entry points unavailable");
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return flykv_fail(KV_ERR_CUDA, "cudaGetDevice failed");
    CUdevice cu = 0;
    NV_TRY(d.device_get(&cu, dev), "cuDeviceGet");
    int attr = 0;
    decltype(&cuDeviceGetAttribute) get_attr = nullptr;
    if (!resolve("cuDeviceGetAttribute", get_attr) || get_attr(&attr, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cu) !=
                                                          CUDA_SUCCESS || !attr)
        return flykv_fail(KV_ERR_CUDA, "device %d reports no multicast support", dev);
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof mp);
    mp.numDevices = (unsigned)n_devices;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = bytes;
    size_t g = 0;
    NV_TRY(d.mc_gran(&g, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
    mp.size = (bytes + g - 1) / g * g;
    if (granularity) *granularity = g;
    CUmemGenericAllocationHandle h;
    CUresult r = d.mc_create(&h, &mp);
    if (r != CUDA_SUCCESS)
        return flykv_fail(KV_ERR_CUDA, "cuMulticastCreate(numDevices=%d, %zu bytes) rejected (%d: %s)", n_devices,
                          (size_t)mp.size, (int)r, errstr(r));
    d.release(h);
    *ok = 1;
    return KV_OK;
}

extern "C" kv_status kv_mc_create(int32_t n_devices, uint64_t bytes, kv_mc** out, int32_t* fd) {
    if (!out || !fd || n_devices < 1 || bytes == 0) return flykv_fail(KV_ERR_INVALID_ARG, "bad kv_mc_create arguments");
    NvlsDrv& d = drv();
    if (!d.mc_ok) return flykv_fail(KV_ERR_CUDA, "multicast driver entry points unavailable");
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof mp);
    mp.numDevices = (unsigned)n_devices;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = bytes;
    size_t g = 0;
    NV_TRY(d.mc_gran(&g, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
    mp.size = (bytes + g - 1) / g * g;
    kv_mc* m = new (std::nothrow) kv_mc();
    if (!m) return flykv_fail(KV_ERR_INVALID_ARG, "out of host memory");
    CUresult r = d.mc_create(&m->h, &mp);
    if (r != CUDA_SUCCESS) {
        delete m;
        return flykv_fail(KV_ERR_CUDA, "cuMulticastCreate failed (%d: %s)", (int)r, errstr(r));
    }
    int f = -1;
    r = d.export_handle(&f, m->h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) {
        d.release(m->h);
        delete m;
        return flykv_fail(KV_ERR_CUDA, "exporting the multicast handle failed (%d: %s)", (int)r, errstr(r));
    }
    m->bytes = mp.size;
    m->n_devices = n_devices;
    *out = m;
    *fd = f;
    return KV_OK;
}

extern "C" kv_status kv_mc_import(int32_t fd, uint64_t bytes, int32_t n_devices, kv_mc** out) {
    if (fd < 0 || !out || bytes == 0) return flykv_fail(KV_ERR_INVALID_ARG, "bad kv_mc_import arguments");
    NvlsDrv& d = drv();
    if (!d.mc_ok) return flykv_fail(KV_ERR_CUDA, "multicast driver entry points unavailable");
    kv_mc* m = new (std::nothrow) kv_mc();
    if (!m) return flykv_fail(KV_ERR_INVALID_ARG, "out of host memory");
    CUresult r = d.import_handle(&m->h, reinterpret_cast<void*>((uintptr_t)fd), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
    if (r != CUDA_SUCCESS) {
        delete m;
        return flykv_fail(KV_ERR_CUDA, "importing the multicast handle failed (%d: %s)", (int)r, errstr(r));
    }
    m->bytes = bytes;
    m->n_devices = n_devices;
    *out = m;
    return KV_OK;
}

extern "C" kv_status kv_mc_add_device(kv_mc* m, int32_t device) {
    if (!m) return flykv_fail(KV_ERR_INVALID_ARG, "multicast object is NULL");
    NvlsDrv& d = drv();
    CUdevice dev;
    NV_TRY(d.device_get(&dev, device), "cuDeviceGet");
    NV_TRY(d.mc_add(m->h, dev), "cuMulticastAddDevice");
    return KV_OK;
}

extern "C" kv_status kv_mc_bind(kv_mc* m, const kv_pool_mem* pool) {
    if (!m || !pool) return flykv_fail(KV_ERR_INVALID_ARG, "bad kv_mc_bind arguments");
    if (pool->bytes > m->bytes)
        return flykv_fail(KV_ERR_INVALID_ARG, "pool of %zu bytes exceeds the multicast object (%zu)", pool->bytes, m->bytes);
    NvlsDrv& d = drv();
    NV_TRY(d.mc_bind(m->h, 0, pool->h, 0, pool->bytes, 0), "cuMulticastBindMem");
    m->bound_device = pool->device;
    m->bound_bytes = pool->bytes;
    return KV_OK;
}

extern "C" kv_status kv_mc_map(kv_mc* m, int32_t device, void** va) {
    if (!m || !va) return flykv_fail(KV_ERR_INVALID_ARG, "bad kv_mc_map arguments");
    NvlsDrv& d = drv();
    CUmulticastObjectProp mp;
    std::memset(&mp, 0, sizeof mp);
    mp.numDevices = (unsigned)m->n_devices;
    mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    mp.size = m->bytes;
    size_t g = 0;
    NV_TRY(d.mc_gran(&g, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity");
    kv_status s = map_rw(d, m->h, m->bytes, g, device, &m->va);
    if (s) return s;
    *va = reinterpret_cast<void*>(m->va);
    return KV_OK;
}

extern "C" kv_status kv_mc_free(kv_mc* m) {
    if (!m) return KV_OK;
    NvlsDrv& d = drv();
    if (m->va) {
        d.unmap(m->va, m->bytes);
        d.addr_free(m->va, m->bytes);
    }
    if (m->bound_device >= 0) {
        CUdevice dev;
        if (d.device_get(&dev, m->bound_device) == CUDA_SUCCESS) d.mc_unbind(m->h, dev, 0, m->bound_bytes);
    }
    d.release(m->h);
    delete m;
    return KV_OK;
}

extern "C" kv_status kv_pool_size(const kv_pool_mem* p, uint64_t* bytes) {
    if (!p || !bytes) return flykv_fail(KV_ERR_INVALID_ARG, "bad kv_pool_size arguments");
    *bytes = p->bytes;
    return KV_OK;
}

extern "C" kv_status kv_mc_size(const kv_mc* m, uint64_t* bytes) {
    if (!m || !bytes) return flykv_fail(KV_ERR_INVALID_ARG, "bad kv_mc_size arguments");
    *bytes = m->bytes;
    return KV_OK;
}

extern "C" kv_status kv_close_fd(int32_t fd) {
    if (fd >= 0) close(fd);
    return KV_OK;
}
