/* probe_mc.c -- does this box's B200 report multicast (NVLS) support? */
#include <stdio.h>
#include <cuda.h>
int main(void) {
    CUdevice d;
    int mc = -1, fabric = -1, n = 0;
    if (cuInit(0) != CUDA_SUCCESS) { printf("cuInit failed\n"); return 1; }
    cuDeviceGetCount(&n);
    cuDeviceGet(&d, 0);
    cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d);
    cuDeviceGetAttribute(&fabric, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d);
    printf("devices=%d multicast_supported=%d fabric_handles=%d\n", n, mc, fabric);
    return 0;
}
