// mc_probe.cu — does this box support NVLink multicast (NVLS, the NVSwitch
// in-switch reduction)?  Prints the driver attributes per device and tries to
// create a multicast object over all visible GPUs (development tool).
#include <cuda.h>
#include <cstdio>

int main() {
  cuInit(0);
  int n = 0;
  cuDeviceGetCount(&n);
  for (int i = 0; i < n; ++i) {
    CUdevice d;
    cuDeviceGet(&d, i);
    int mc = -1, fab = -1, vmm = -1;
    cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d);
    cuDeviceGetAttribute(&vmm, CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED, d);
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, d);
    printf("dev %d: multicast=%d vmm=%d fabric_handle=%d\n", i, mc, vmm, fab);
  }
  CUmulticastObjectProp p = {};
  p.numDevices = n;
  p.size = 2ull << 20;
  p.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  CUresult r = cuMulticastGetGranularity(&gran, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  printf("cuMulticastGetGranularity: %d gran=%zu\n", (int)r, gran);
  if (gran) p.size = gran;
  CUmemGenericAllocationHandle h;
  r = cuMulticastCreate(&h, &p);
  printf("cuMulticastCreate(%d devices): %d\n", n, (int)r);
  return 0;
}
