// Probe: NVLS multicast on this lease through the CUDA driver API (no IPC handle export):
// create a multicast object for the visible device(s), bind physical memory, map the multicast
// VA, and run multimem.red.add.f32 / multimem.ld_reduce from a kernel. Prints each step.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); printf("FAIL %s: %s\n", #x, s); return 1; } else printf("ok   %s\n", #x); } while (0)
__global__ void red_kernel(float* mc, float* uc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    float v = float(i % 7);
    asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(mc + i), "f"(v) : "memory");
  }
}
__global__ void red_v4_kernel(float* mc, int n4) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n4) {
    asm volatile("multimem.red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 4 * i), "f"(1.f), "f"(2.f), "f"(3.f), "f"(4.f) : "memory");
  }
}
int main() {
  CK(cuInit(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  int mcs = 0; CK(cuDeviceGetAttribute(&mcs, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("multicast supported attribute: %d\n", mcs);
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  size_t n = 1 << 20, bytes = n * 4;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.size = bytes;
  size_t gran = 0, gmin = 0;
  CUmemGenericAllocationHandle mch;
  const unsigned long long types[3] = {0ull, (unsigned long long)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                       (unsigned long long)CU_MEM_HANDLE_TYPE_FABRIC};
  int ok = 0;
  for (int t = 0; t < 3 && !ok; ++t) {
    mp.handleTypes = types[t];
    mp.size = bytes;
    if (cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS) { printf("gran min fail t=%d\n", t); continue; }
    cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    mp.size = (bytes + gmin - 1) / gmin * gmin;
    CUresult r = cuMulticastCreate(&mch, &mp);
    const char* es; cuGetErrorString(r, &es);
    printf("handleTypes %llu: min gran %zu rec %zu size %zu -> cuMulticastCreate %s\n", types[t], gmin, gran, mp.size, es);
    ok = r == CUDA_SUCCESS;
  }
  if (!ok) return 1;
  gran = gmin;
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ap.location.id = dev;
  ap.requestedHandleTypes = (CUmemAllocationHandleType)mp.handleTypes;
  size_t ag = 0; CK(cuMemGetAllocationGranularity(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CUmemGenericAllocationHandle ph; CK(cuMemCreate(&ph, mp.size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, ph, 0, mp.size, 0));
  CUdeviceptr uva, mva;
  CK(cuMemAddressReserve(&uva, mp.size, gran, 0, 0)); CK(cuMemMap(uva, mp.size, 0, ph, 0));
  CK(cuMemAddressReserve(&mva, mp.size, gran, 0, 0)); CK(cuMemMap(mva, mp.size, 0, mch, 0));
  CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = dev; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uva, mp.size, &ad, 1)); CK(cuMemSetAccess(mva, mp.size, &ad, 1));
  cudaMemset((void*)uva, 0, bytes);
  red_kernel<<<(n + 255) / 256, 256>>>((float*)mva, (float*)uva, int(n));
  red_kernel<<<(n + 255) / 256, 256>>>((float*)mva, (float*)uva, int(n));
  red_v4_kernel<<<(n / 4 + 255) / 256, 256>>>((float*)mva, int(n / 4));
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernels: %s\n", cudaGetErrorString(e));
  float h[8]; cudaMemcpy(h, (void*)uva, sizeof(h), cudaMemcpyDeviceToHost);
  printf("values: "); for (int i = 0; i < 8; ++i) printf("%g ", h[i]); printf("  (want 2*(i%%7) + {1,2,3,4})\n");
  return 0;
}
