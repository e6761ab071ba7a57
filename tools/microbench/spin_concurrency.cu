// Probe (not product code): can a 1-thread spin kernel on stream A wait for work queued on
// stream B of the same process when B runs a persistent, smem-heavy grid first?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(volatile unsigned* flag, unsigned* out) {
  long long t0 = clock64();
  while (*flag == 0) { if (clock64() - t0 > 4000000000ll) { out[0] = 1; return; } __nanosleep(256); }
  out[0] = 2;
}
__global__ void big(unsigned* sink) {
  extern __shared__ unsigned sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  unsigned a = 0;
  for (int i = 0; i < 20000; i++) a += sm[(threadIdx.x + i) & 127];
  if (a == 7) sink[0] = a;
}
__global__ void nosmem(unsigned* sink) {
  unsigned a = threadIdx.x;
  for (int i = 0; i < 20000; i++) a = a * 3 + 1;
  if (a == 7) sink[0] = a;
}
__global__ void setflag(unsigned* flag) { *flag = 1; __threadfence_system(); }
int main(int argc, char** argv) {
  const int smem = argc > 1 ? atoi(argv[1]) : 45000;
  unsigned *flag, *out, *sink;
  cudaMalloc(&flag, 4); cudaMalloc(&out, 4); cudaMalloc(&sink, 4);
  cudaMemset(flag, 0, 4); cudaMemset(out, 0, 4);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  int ck; cudaDeviceGetAttribute(&ck, cudaDevAttrConcurrentKernels, 0);
  printf("concurrentKernels=%d\n", ck);
  if (argc > 2) {   // reverse: the setter first, then the spinner
    setflag<<<1, 1, 0, b>>>(flag);
    spin<<<1, 1, 0, a>>>(flag, out);
    cudaDeviceSynchronize();
    unsigned r; cudaMemcpy(&r, out, 4, cudaMemcpyDeviceToHost);
    printf("reverse order: spin result %u\n", r);
    cudaMemset(flag, 0, 4); cudaMemset(out, 0, 4);
    // two spinners on separate streams setting each other's flag
    return 0;
  }
  spin<<<1, 1, 0, a>>>(flag, out);
  if (smem) big<<<nsm * 5, 128, smem, b>>>(sink);
  else nosmem<<<nsm * 5, 128, 0, b>>>(sink);
  setflag<<<1, 1, 0, b>>>(flag);
  cudaDeviceSynchronize();
  unsigned r; cudaMemcpy(&r, out, 4, cudaMemcpyDeviceToHost);
  printf("smem %d: spin result %u (2 = saw the flag, 1 = timed out): %s\n", smem, r, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
