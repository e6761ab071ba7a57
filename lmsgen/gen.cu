// lmsgen CUDA generator — INPUT GENERATION ONLY (no method arithmetic).
//
// Byte-identical device implementation of lmsgen/__init__.py (SURVEY.md Appendix A recipe):
// counter-based SplitMix64 draws r(seed, tag, t, i, f), u(x, n) = (x * n) >> 64, LR records
// of exactly 70 B and CM task_events lines of 130..145 B.  Used by tests and bench.py to
// build 10M-record micro-batches in HBM; pinned against the Python generator by tests.
#include <cuda_runtime.h>
#include <cub/device/device_scan.cuh>

#include <cstdint>

namespace {

constexpr uint64_t kTagLR = 1, kTagCM = 2, kTagKey = 4;

__host__ __device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t u(uint64_t x, uint64_t n) { return __umul64hi(x, n); }
__host__ __device__ __forceinline__ uint64_t rdraw(uint64_t seed, uint64_t tag, uint64_t t, uint64_t i,
                                                   uint64_t f) {
  return mix(mix(mix(mix(mix(seed) ^ tag) ^ t) ^ i) ^ f);
}

__device__ __forceinline__ int ndigits(uint64_t v) {
  int n = 1;
  while (v >= 10) { v /= 10; n++; }
  return n;
}
__device__ __forceinline__ void put_pad(uint8_t* p, uint64_t v, int w) {
  for (int k = w - 1; k >= 0; k--) { p[k] = (uint8_t)('0' + v % 10); v /= 10; }
}
__device__ __forceinline__ int put_dec(uint8_t* p, uint64_t v) {
  const int n = ndigits(v);
  put_pad(p, v, n);
  return n;
}

__global__ void k_lr(uint64_t seed, uint64_t t, uint64_t count, uint64_t H, uint64_t V, uint8_t* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t sp = mix(mix(mix(seed) ^ kTagLR) ^ t);
  const uint64_t rp = mix(sp ^ i);
  const uint64_t vid = u(mix(rp ^ 0), V), xway = u(mix(rp ^ 1), H), d = u(mix(rp ^ 2), 2);
  const uint64_t seg = u(mix(rp ^ 3), 100), lane = u(mix(rp ^ 4), 5);
  const uint64_t k = (xway * 2 + d) * 100 + seg;
  const int64_t mu = 10 + (int64_t)u(rdraw(seed, kTagKey, 0, k, 0), 81);
  int64_t spd = mu + (int64_t)u(mix(rp ^ 5), 21) - 10;
  spd = spd < 0 ? 0 : (spd > 100 ? 100 : spd);
  const uint64_t pos = seg * 5280 + u(mix(rp ^ 6), 5280);
  uint8_t b[70];
  // Type(1),Time(6),VID(10),Spd(3),XWay(3),Lane(1),Dir(1),Seg(3),Pos(8),QID(8),Sinit(2),Send(2),DOW(1),TOD(4),Day(2)\n
  int o = 0;
  auto fld = [&](uint64_t v, int w, char sep) { put_pad(b + o, v, w); o += w; b[o++] = (uint8_t)sep; };
  fld(0, 1, ','); fld(t, 6, ','); fld(vid, 10, ','); fld((uint64_t)spd, 3, ','); fld(xway, 3, ',');
  fld(lane, 1, ','); fld(d, 1, ','); fld(seg, 3, ','); fld(pos, 8, ','); fld(0, 8, ',');
  fld(0, 2, ','); fld(0, 2, ','); fld(0, 1, ','); fld(0, 4, ','); fld(0, 2, '\n');
  uint8_t* dst = out + i * 70;
  for (int j = 0; j < 70; j++) dst[j] = b[j];
}

__global__ void k_cm_len(uint64_t seed, uint64_t t, uint64_t count, uint32_t* len) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t rp = mix(mix(mix(mix(seed) ^ kTagCM) ^ t) ^ i);
  len[i] = 130 + (uint32_t)u(mix(rp ^ 0), 16);
}

__global__ void k_cm(uint64_t seed, uint64_t t, uint64_t count, uint64_t J, int64_t sel_ppm,
                     const uint64_t* off, const uint32_t* len, uint8_t* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t rp = mix(mix(mix(mix(seed) ^ kTagCM) ^ t) ^ i);
  auto rr = [&](uint64_t f) { return mix(rp ^ f); };
  const uint32_t L = len[i];
  const uint64_t j = u(rr(1), J);
  const uint64_t job = 1000000000ull + u(rdraw(seed, kTagKey, 0, j, 1), 9000000000ull);
  const uint64_t task = u(rr(2), 10000);
  const uint64_t machine = 1 + u(rr(3), 6000000000ull);
  uint64_t ev;
  if (sel_ppm < 0) {
    const uint64_t e = u(rr(4), 100);
    const uint64_t thr[9] = {26, 52, 54, 56, 78, 96, 97, 99, 100};
    ev = 0;
    while (e >= thr[ev]) ev++;
  } else {
    if (u(rr(4), 1000000) < (uint64_t)sel_ppm) ev = 1;
    else { const uint64_t o8[8] = {0, 2, 3, 4, 5, 6, 7, 8}; ev = o8[u(rr(11), 8)]; }
  }
  const uint64_t cat = u(rr(5), 4), prio = u(rr(6), 12);
  const uint64_t cpu = 1 + u(rr(7), 500000), ram = 1 + u(rr(8), 500000), disk = 1 + u(rr(9), 500000);
  const uint64_t cons = u(rr(10), 2);
  uint8_t* p = out + off[i];
  int o = 0;
  o += put_dec(p + o, t); p[o++] = ','; p[o++] = ',';
  o += put_dec(p + o, job); p[o++] = ',';
  o += put_dec(p + o, task); p[o++] = ',';
  o += put_dec(p + o, machine); p[o++] = ',';
  o += put_dec(p + o, ev); p[o++] = ',';
  const int tail = 33 + ndigits(prio);
  const int ulen = (int)L - o - tail;
  const char* B64 = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/";
  for (int c = 0; c < ulen; c++) p[o++] = (uint8_t)B64[u(rr(16 + c), 64)];
  p[o++] = ','; o += put_dec(p + o, cat);
  p[o++] = ','; o += put_dec(p + o, prio);
  p[o++] = ','; p[o++] = '0'; p[o++] = '.'; put_pad(p + o, cpu, 6); o += 6;
  p[o++] = ','; p[o++] = '0'; p[o++] = '.'; put_pad(p + o, ram, 6); o += 6;
  p[o++] = ','; p[o++] = '0'; p[o++] = '.'; put_pad(p + o, disk, 6); o += 6;
  p[o++] = ','; o += put_dec(p + o, cons);
  p[o++] = '\n';
}

}  // namespace

extern "C" {

// LR second t: count records (count * 70 bytes) into out (device).  Returns a cudaError_t.
int lmsgen_lr_second(uint64_t seed, uint64_t t, uint64_t count, uint64_t num_xways, uint64_t num_vehicles,
                     void* out, void* stream) {
  if (count == 0) return 0;
  k_lr<<<(unsigned)((count + 255) / 256), 256, 0, (cudaStream_t)stream>>>(seed, t, count, num_xways,
                                                                          num_vehicles, (uint8_t*)out);
  return (int)cudaGetLastError();
}

// CM second t: count records into out (device, capacity >= 145 * count).  *nbytes_out = bytes
// written (synchronous: the host needs the size).  sel_ppm < 0: default eventType mix.
int lmsgen_cm_second(uint64_t seed, uint64_t t, uint64_t count, uint64_t num_jobs, int64_t sel_ppm,
                     void* out, uint64_t* nbytes_out, void* stream) {
  *nbytes_out = 0;
  if (count == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t* len = nullptr;
  uint64_t* off = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  cudaError_t e;
  if ((e = cudaMallocAsync(&len, (count + 1) * sizeof(uint32_t), st))) return (int)e;
  if ((e = cudaMallocAsync(&off, (count + 1) * sizeof(uint64_t), st))) return (int)e;
  k_cm_len<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(seed, t, count, len);
  cudaMemsetAsync(len + count, 0, sizeof(uint32_t), st);
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, len, off, count + 1, st);
  if ((e = cudaMallocAsync(&tmp, tmp_bytes, st))) return (int)e;
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, len, off, count + 1, st);
  k_cm<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(seed, t, count, num_jobs, sel_ppm, off, len,
                                                         (uint8_t*)out);
  uint64_t total = 0;
  cudaMemcpyAsync(&total, off + count, sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(tmp, st);
  cudaFreeAsync(len, st);
  cudaFreeAsync(off, st);
  if ((e = cudaStreamSynchronize(st))) return (int)e;
  *nbytes_out = total;
  return (int)cudaGetLastError();
}

}  // extern "C"
