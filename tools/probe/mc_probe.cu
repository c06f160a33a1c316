// Probe: can this process create a CUDA multicast object (NVLS) at all?
#include <cstdio>
#include <cuda.h>
int main() {
  cuInit(0);
  CUdevice dev; cuDeviceGet(&dev, 0);
  CUcontext ctx; cuDevicePrimaryCtxRetain(&ctx, dev); cuCtxSetCurrent(ctx);
  int mc = 0; cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  printf("multicast supported attr = %d\n", mc);
  for (int ht : {0, (int)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, (int)CU_MEM_HANDLE_TYPE_FABRIC}) {
    CUmulticastObjectProp p = {};
    p.numDevices = 1; p.handleTypes = ht; p.size = 2 << 20; p.flags = 0;
    size_t g = 0;
    CUresult e0 = cuMulticastGetGranularity(&g, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    CUmemGenericAllocationHandle h;
    CUresult e = cuMulticastCreate(&h, &p);
    const char* s = nullptr; cuGetErrorString(e, &s);
    printf("handleTypes=%d gran=%zu (%d) create -> %d %s\n", ht, g, (int)e0, (int)e, s ? s : "");
  }
  return 0;
}
