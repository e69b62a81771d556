// Probe: is an NVLS multicast object usable with the GPU(s) visible here?
// nvcc -arch=sm_100a -o /tmp/nvls_probe scripts/probe/nvls_probe.cu -lcuda
#include <cuda.h>
#include <cstdio>
#include <cstdint>
#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
  printf("%s -> %d %s\n", #x, (int)r, s); return 1; } } while (0)

__global__ void mc_store(uint32_t* mc, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) asm volatile("multimem.st.relaxed.sys.global.u32 [%0], %1;" ::"l"(mc + i), "r"(i * 3u) : "memory");
}
__global__ void mc_ldred(const float* mc, float* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { float v; asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=f"(v) : "l"(mc + i) : "memory"); out[i] = v; }
}

int main() {
  CK(cuInit(0));
  int ndev; CK(cuDeviceGetCount(&ndev));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  int mc = 0; CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  printf("devices=%d multicast_supported=%d\n", ndev, mc);
  if (!mc) return 0;
  CUcontext ctx; CK(cuDevicePrimaryCtxRetain(&ctx, dev)); CK(cuCtxSetCurrent(ctx));
  CUmulticastObjectProp prop = {};
  prop.numDevices = 1; prop.size = 2 << 20; prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0; CK(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  prop.size = ((prop.size + gran - 1) / gran) * gran;
  printf("granularity=%zu size=%zu\n", gran, prop.size);
  CUmemGenericAllocationHandle mch;
  {
    CUresult r = CUDA_ERROR_UNKNOWN;
    unsigned long long hts[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0, CU_MEM_HANDLE_TYPE_FABRIC};
    for (int t = 0; t < 3 && r != CUDA_SUCCESS; ++t) {
      prop.handleTypes = hts[t];
      r = cuMulticastCreate(&mch, &prop);
      printf("cuMulticastCreate(numDevices=1, handleTypes=%llu) -> %d\n", hts[t], (int)r);
    }
    if (r != CUDA_SUCCESS) return 1;
  }
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {}; ap.type = CU_MEM_ALLOCATION_TYPE_PINNED; ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0; ap.requestedHandleTypes = (CUmemAllocationHandleType)prop.handleTypes;
  CUmemGenericAllocationHandle mem; CK(cuMemCreate(&mem, prop.size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, mem, 0, prop.size, 0));
  CUdeviceptr uc, mcp;
  CK(cuMemAddressReserve(&uc, prop.size, gran, 0, 0)); CK(cuMemMap(uc, prop.size, 0, mem, 0));
  CK(cuMemAddressReserve(&mcp, prop.size, gran, 0, 0)); CK(cuMemMap(mcp, prop.size, 0, mch, 0));
  CUmemAccessDesc ad = {}; ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE; ad.location.id = 0; ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, prop.size, &ad, 1)); CK(cuMemSetAccess(mcp, prop.size, &ad, 1));
  int n = 1 << 16;
  mc_store<<<n / 256, 256>>>((uint32_t*)mcp, n);
  CK(cuCtxSynchronize());
  uint32_t h[4]; CK(cuMemcpyDtoH(h, uc + 4 * 100, 16));
  printf("multimem.st via NVLS -> unicast[100..103] = %u %u %u %u (want 300 303 306 309)\n", h[0], h[1], h[2], h[3]);
  float* out; cudaMalloc(&out, n * 4);
  float ones[4] = {1.5f, 2.5f, 3.5f, 4.5f}; CK(cuMemcpyHtoD(uc, ones, 16));
  mc_ldred<<<n / 256, 256>>>((const float*)mcp, out, n);
  CK(cuCtxSynchronize());
  float o[4]; cudaMemcpy(o, out, 16, cudaMemcpyDeviceToHost);
  printf("multimem.ld_reduce -> %g %g %g %g (one device: the values themselves)\n", o[0], o[1], o[2], o[3]);
  return 0;
}
