// probe_mc2.cu -- which cuMulticastCreate arguments does this box accept?
// numDevices 1 and 2, sizes of one minimum / one recommended granule and
// 4 GiB, handle types none / posix_fd / fabric; prints every result.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probe_mc2 scripts/probe_mc2.cu -lcuda
#include <cstdio>
#include <cstring>
#include <cuda.h>
#include <cuda_runtime.h>

int main() {
    cudaSetDevice(0);
    cudaFree(0);
    cuInit(0);
    CUdevice dev;
    cuDeviceGet(&dev, 0);
    int mcs = 0, fab = 0, vmm = 0, ndev = 0;
    cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, dev);
    cuDeviceGetCount(&ndev);
    int drv = 0;
    cuDriverGetVersion(&drv);
    printf("driver %d devices %d multicast %d fabric %d vmm %d\n", drv, ndev, mcs, fab, vmm);
    const struct { CUmemAllocationHandleType t; const char* name; } kinds[] = {
        {CU_MEM_HANDLE_TYPE_NONE, "none"}, {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, "posix_fd"},
        {CU_MEM_HANDLE_TYPE_FABRIC, "fabric"}};
    for (int nd : {1, 2}) {
        for (const auto& k : kinds) {
            CUmulticastObjectProp mp;
            std::memset(&mp, 0, sizeof(mp));
            mp.numDevices = nd;
            mp.handleTypes = k.t;
            mp.size = 2 << 20;
            size_t gmin = 0, grec = 0;
            CUresult g1 = cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM);
            CUresult g2 = cuMulticastGetGranularity(&grec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
            for (size_t sz : {gmin, grec, (size_t)4 << 30}) {
                if (!sz) continue;
                mp.size = sz;
                CUmemGenericAllocationHandle mc;
                CUresult r = cuMulticastCreate(&mc, &mp);
                const char* es = "";
                cuGetErrorString(r, &es);
                printf("numDevices=%d handle=%-8s gran(min %zu rc %d, rec %zu rc %d) size=%zu -> %d %s\n", nd, k.name,
                       gmin, (int)g1, grec, (int)g2, sz, (int)r, es);
                if (r == CUDA_SUCCESS) {
                    CUresult a = cuMulticastAddDevice(mc, dev);
                    cuGetErrorString(a, &es);
                    printf("    AddDevice -> %d %s\n", (int)a, es);
                    cuMemRelease(mc);
                }
            }
        }
    }
    return 0;
}
