// Design-probe microbenchmarks for the LMStream B200 hot path (not product code).
// Measures: bulk-copy (TMA 1D) streaming read, LDG.128 streaming read,
// shared-memory u32 atomic throughput (random keys in a 2000-entry table),
// global RED throughput on an L2-resident table, and __match_any_sync cost.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(b)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" :: "r"(smem_u32(b)), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b)) : "memory");
}

template <int STAGES, int TILE>
__global__ void k_bulk_read(const uint8_t* __restrict__ src, size_t nbytes, unsigned long long* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t full[STAGES];
  size_t ntiles = nbytes / TILE;
  if (threadIdx.x == 0) { for (int s = 0; s < STAGES; s++) mbar_init(&full[s], 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  size_t first = blockIdx.x;
  uint32_t acc = 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; s++) {
      size_t t = first + (size_t)s * gridDim.x;
      if (t < ntiles) { mbar_expect_tx(&full[s], TILE); bulk_g2s(sm + s * TILE, src + t * TILE, TILE, &full[s]); }
    }
  }
  int it = 0;
  for (size_t t = first; t < ntiles; t += gridDim.x, it++) {
    int s = it % STAGES; uint32_t ph = (it / STAGES) & 1;
    mbar_wait(&full[s], ph);
    const uint32_t* w = (const uint32_t*)(sm + s * TILE);
    for (int i = threadIdx.x; i < TILE / 4; i += blockDim.x) acc ^= w[i];
    __syncthreads();
    if (threadIdx.x == 0) {
      size_t tn = t + (size_t)STAGES * gridDim.x;
      if (tn < ntiles) { mbar_expect_tx(&full[s], TILE); bulk_g2s(sm + s * TILE, src + tn * TILE, TILE, &full[s]); }
    }
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

__global__ void k_ldg_read(const int4* __restrict__ src, size_t n16, unsigned long long* out) {
  uint32_t acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n16; i += 4 * stride) {
    int4 a = __ldg(src + i), b = __ldg(src + i + stride), c = __ldg(src + i + 2 * stride), d = __ldg(src + i + 3 * stride);
    acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
  }
  for (; i < n16; i += stride) { int4 a = __ldg(src + i); acc ^= a.x ^ a.y ^ a.z ^ a.w; }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }

// Each thread does ITERS atomics into a per-CTA table of K u32 entries.
template <bool RET>
__global__ void k_atoms(int iters, int K, unsigned long long* out) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < K; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t seed = hash32(blockIdx.x * 1024 + threadIdx.x);
  uint32_t acc = 0;
  for (int i = 0; i < iters; i++) {
    seed = seed * 1664525u + 1013904223u;
    uint32_t k = __umulhi(seed, (uint32_t)K);
    if (RET) acc += atomicAdd(&tab[k], (1u << 22) | (seed & 127));
    else atomicAdd(&tab[k], (1u << 22) | (seed & 127));
  }
  __syncthreads();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < K; i += blockDim.x) s += tab[i];
  if ((s ^ acc) == 0x12345678u) atomicAdd(out, 1ull);
}

// Non-atomic baseline: LDS+STS RMW (racy, only for throughput comparison)
__global__ void k_lds_rmw(int iters, int K, unsigned long long* out) {
  extern __shared__ uint32_t tab[];
  for (int i = threadIdx.x; i < K; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t seed = hash32(blockIdx.x * 1024 + threadIdx.x);
  for (int i = 0; i < iters; i++) {
    seed = seed * 1664525u + 1013904223u;
    uint32_t k = __umulhi(seed, (uint32_t)K);
    volatile uint32_t* t = tab;
    t[k] = t[k] + ((1u << 22) | (seed & 127));
  }
  __syncthreads();
  uint32_t s = 0;
  for (int i = threadIdx.x; i < K; i += blockDim.x) s += tab[i];
  if (s == 0x12345678u) atomicAdd(out, 1ull);
}

__global__ void k_redg(int iters, uint32_t K, unsigned long long* tab, unsigned long long* out) {
  uint32_t seed = hash32(blockIdx.x * 1024 + threadIdx.x);
  for (int i = 0; i < iters; i++) {
    seed = seed * 1664525u + 1013904223u;
    uint32_t k = __umulhi(seed, K);
    atomicAdd(&tab[k], (unsigned long long)(seed & 1023));
  }
}

__global__ void k_match(int iters, unsigned long long* out) {
  uint32_t seed = hash32(blockIdx.x * 1024 + threadIdx.x);
  uint32_t acc = 0;
  for (int i = 0; i < iters; i++) {
    seed = seed * 1664525u + 1013904223u;
    acc += __match_any_sync(0xffffffffu, (unsigned long long)(seed >> 20));
  }
  if (acc == 0x12345678u) atomicAdd(out, 1ull);
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("gpu %s sms %d smem/blk optin %zu l2 %d MB clock %d kHz\n", p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.l2CacheSize >> 20, p.clockRate);
  int nsm = p.multiProcessorCount;
  size_t nbytes = (size_t)4 << 30;
  uint8_t* buf; CK(cudaMalloc(&buf, nbytes)); CK(cudaMemset(buf, 1, nbytes));
  unsigned long long* out; CK(cudaMalloc(&out, 1 << 20)); CK(cudaMemset(out, 0, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // LDG read
  for (int bpsm : {4, 8, 16}) {
    int grid = nsm * bpsm;
    k_ldg_read<<<grid, 256>>>((const int4*)buf, nbytes / 16, out);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; r++) k_ldg_read<<<grid, 256>>>((const int4*)buf, nbytes / 16, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("ldg_read grid=%d: %.1f GB/s\n", grid, 5.0 * nbytes / (ms * 1e-3) / 1e9);
  }
  // bulk read
#define BULK(ST, TL, BPSM, THR) { \
    auto kf = k_bulk_read<ST, TL>; int sm = ST * TL; \
    CK(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
    int grid = nsm * BPSM; kf<<<grid, THR, sm>>>(buf, nbytes, out); CK(cudaGetLastError()); \
    cudaEventRecord(e0); for (int r = 0; r < 5; r++) kf<<<grid, THR, sm>>>(buf, nbytes, out); \
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1); \
    printf("bulk_read stages=%d tile=%d ctas/sm=%d thr=%d: %.1f GB/s\n", ST, TL, BPSM, THR, 5.0 * nbytes / (ms * 1e-3) / 1e9); }
  BULK(4, 16384, 1, 256) BULK(4, 16384, 2, 256) BULK(6, 16384, 2, 256) BULK(3, 32768, 2, 256)
  BULK(4, 17920, 2, 128) BULK(4, 8192, 4, 128) BULK(8, 8192, 2, 256) BULK(2, 32768, 3, 256)
  // smem atomics
  for (int K : {2000, 4096}) for (int thr : {256, 512}) {
    int iters = 4096; int grid = nsm * (1024 / thr) * 2;
    k_atoms<false><<<grid, thr, K * 4>>>(iters, K, out);
    cudaEventRecord(e0); k_atoms<false><<<grid, thr, K * 4>>>(iters, K, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * thr * iters;
    printf("atoms_noret K=%d thr=%d: %.2f Gop/s = %.3f SM-cycles/op @%.0fMHz\n", K, thr, ops / (ms * 1e-3) / 1e9,
           (ms * 1e-3) * p.clockRate * 1e3 * nsm / ops, p.clockRate / 1e3);
    k_atoms<true><<<grid, thr, K * 4>>>(iters, K, out);
    cudaEventRecord(e0); k_atoms<true><<<grid, thr, K * 4>>>(iters, K, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("atoms_ret   K=%d thr=%d: %.2f Gop/s\n", K, thr, ops / (ms * 1e-3) / 1e9);
    k_lds_rmw<<<grid, thr, K * 4>>>(iters, K, out);
    cudaEventRecord(e0); k_lds_rmw<<<grid, thr, K * 4>>>(iters, K, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    printf("lds_rmw     K=%d thr=%d: %.2f Gop/s\n", K, thr, ops / (ms * 1e-3) / 1e9);
  }
  // global RED
  unsigned long long* gt; CK(cudaMalloc(&gt, 64 << 20)); CK(cudaMemset(gt, 0, 64 << 20));
  for (uint32_t K : {4u, 100u, 2000u, 16384u, 1u << 20}) {
    int iters = 256; int grid = nsm * 8, thr = 256;
    k_redg<<<grid, thr>>>(iters, K, gt, out);
    cudaEventRecord(e0); k_redg<<<grid, thr>>>(iters, K, gt, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * thr * iters;
    printf("redg_u64 K=%u: %.2f Gop/s\n", K, ops / (ms * 1e-3) / 1e9);
  }
  {
    int iters = 4096; int grid = nsm * 8, thr = 256;
    k_match<<<grid, thr>>>(iters, out);
    cudaEventRecord(e0); k_match<<<grid, thr>>>(iters, out); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * thr * iters / 32;
    printf("match_any_u64: %.2f G warp-ops/s = %.2f SM-cycles per warp-op\n", ops / (ms * 1e-3) / 1e9,
           (ms * 1e-3) * p.clockRate * 1e3 * nsm / ops);
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
