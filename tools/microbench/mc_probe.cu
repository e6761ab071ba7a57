// Probe: does this box's GPU support NVLink-switch multicast (NVLS) objects, and do multimem
// reductions work on a multicast group of the visible devices?  (f1 groundwork: the dense LR2 /
// CM1 merge tables reduced in the switch with multimem.red instead of an owner exchange.)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o mc_probe mc_probe.cu -lcuda && ./mc_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    CUresult r_ = (x);                                                                 \
    if (r_ != CUDA_SUCCESS) {                                                          \
      const char* s_ = nullptr;                                                        \
      cuGetErrorString(r_, &s_);                                                       \
      printf("FAIL %s: %d %s\n", #x, (int)r_, s_ ? s_ : "?");                          \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

__global__ void k_red(unsigned long long* mc, int n, unsigned long long add) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(mc + i), "l"(add) : "memory");
}
__global__ void k_ldred(const unsigned long long* mc, unsigned long long* out, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    unsigned long long v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.u64 %0, [%1];" : "=l"(v) : "l"(mc + i) : "memory");
    out[i] = v;
  }
}

int main() {
  CK(cuInit(0));
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  printf("devices %d\n", ndev);
  for (int d = 0; d < ndev; d++) {
    CUdevice dev;
    CK(cuDeviceGet(&dev, d));
    int mc = 0, fab = 0;
    CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
    printf("device %d: multicast supported %d, fabric handles %d\n", d, mc, fab);
  }
  CUdevice dev0;
  CK(cuDeviceGet(&dev0, 0));
  CUcontext ctx;
  CK(cuDevicePrimaryCtxRetain(&ctx, dev0));
  CK(cuCtxSetCurrent(ctx));
  const int n = 1 << 16;
  CUmulticastObjectProp prop = {};
  CUmemGenericAllocationHandle mch = 0;
  size_t gran = 0;
  CUmemAllocationHandleType chosen = CU_MEM_HANDLE_TYPE_NONE;
  const CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                              CU_MEM_HANDLE_TYPE_FABRIC};
  bool made = false;
  for (int ti = 0; ti < 3 && !made; ti++) {
    prop = {};
    prop.numDevices = 1;
    prop.size = (size_t)n * 8;
    prop.handleTypes = types[ti];
    CUresult r = cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    if (r != CUDA_SUCCESS) { printf("granularity(type %d): %d\n", (int)types[ti], (int)r); continue; }
    prop.size = (prop.size + gran - 1) / gran * gran;
    r = cuMulticastCreate(&mch, &prop);
    printf("cuMulticastCreate(handle type %d, size %zu, gran %zu): %d\n", (int)types[ti], prop.size, gran, (int)r);
    if (r == CUDA_SUCCESS) { made = true; chosen = types[ti]; }
  }
  if (!made) { printf("no multicast object could be created\n"); return 1; }
  CK(cuMulticastAddDevice(mch, dev0));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = chosen;
  size_t pg = 0;
  CK(cuMemGetAllocationGranularity(&pg, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  const size_t sz = (prop.size + pg - 1) / pg * pg;
  CUmemGenericAllocationHandle ph;
  CK(cuMemCreate(&ph, sz, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, ph, 0, sz, 0));
  CUdeviceptr uc = 0, mcp = 0;
  CK(cuMemAddressReserve(&uc, sz, 0, 0, 0));
  CK(cuMemMap(uc, sz, 0, ph, 0));
  CK(cuMemAddressReserve(&mcp, prop.size, 0, 0, 0));
  CK(cuMemMap(mcp, prop.size, 0, mch, 0));
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, sz, &acc, 1));
  CK(cuMemSetAccess(mcp, prop.size, &acc, 1));
  cudaMemset((void*)uc, 0, (size_t)n * 8);
  k_red<<<64, 256>>>((unsigned long long*)mcp, n, 3ull);
  k_red<<<64, 256>>>((unsigned long long*)mcp, n, 4ull);
  unsigned long long* out = nullptr;
  cudaMalloc(&out, (size_t)n * 8);
  k_ldred<<<64, 256>>>((const unsigned long long*)mcp, out, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernels: %s\n", cudaGetErrorString(e));
  std::vector<unsigned long long> h(n), hu(n);
  cudaMemcpy(h.data(), out, (size_t)n * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(hu.data(), (void*)uc, (size_t)n * 8, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n; i++) bad += (h[i] != 7ull) + (hu[i] != 7ull);
  printf("multimem.red + ld_reduce on a 1-device group: %s (%d mismatches)\n", bad ? "WRONG" : "ok", bad);
  return 0;
}
