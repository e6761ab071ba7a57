// Pipe-mix probe (not product code): throughput of integer op mixes per SM, to decide how
// to balance the CM pass-1 byte classification between the ALU and FMA pipes on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NCH 8
template <int MIX>
__global__ void k(uint32_t* out, uint32_t seed, uint32_t one, int iters) {
  uint32_t x[NCH];
#pragma unroll
  for (int c = 0; c < NCH; c++) x[c] = seed + threadIdx.x * 7 + c;
  const uint32_t K1 = seed ^ 0x7F7F7F7Fu, K2 = seed ^ 0x2C2C2C2Cu;   // runtime constants
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int c = 0; c < NCH; c++) {
      uint32_t v = x[c];
      if (MIX == 0) {                    // 4 x LOP3
        asm("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v) : "r"(K1), "r"(K2));
      } else if (MIX == 1) {             // 4 x add (VIADD / IADD3)
        asm("add.u32 %0, %0, %1;" : "+r"(v) : "r"(K1));
        asm("add.u32 %0, %0, %1;" : "+r"(v) : "r"(K2));
        asm("add.u32 %0, %0, %1;" : "+r"(v) : "r"(K1));
        asm("add.u32 %0, %0, %1;" : "+r"(v) : "r"(K2));
      } else if (MIX == 2) {             // 4 x IMAD (runtime multiplier)
        asm("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(one), "r"(K1));
        asm("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(one), "r"(K2));
        asm("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(one), "r"(K1));
        asm("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(one), "r"(K2));
      } else if (MIX == 3) {             // 4 x dp4a
        asm("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(K2), "r"(K1));
        asm("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(K2), "r"(K1));
      } else if (MIX == 4) {             // 2 LOP3 + 2 add
        asm("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("add.u32 %0, %0, %1;" : "+r"(v) : "r"(K1));
        asm("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("add.u32 %0, %0, %1;" : "+r"(v) : "r"(K2));
      } else if (MIX == 5) {             // 2 LOP3 + 2 IMAD
        asm("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(one), "r"(K1));
        asm("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(one), "r"(K2));
      } else if (MIX == 6) {             // 2 LOP3 + 2 dp4a
        asm("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("lop3.b32 %0, %0, %1, %2, 0x6a;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("dp4a.u32.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(K2), "r"(K1));
      } else if (MIX == 7) {             // 2 add + 2 IMAD
        asm("add.u32 %0, %0, %1;" : "+r"(v) : "r"(K1));
        asm("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(one), "r"(K1));
        asm("add.u32 %0, %0, %1;" : "+r"(v) : "r"(K2));
        asm("mad.lo.u32 %0, %0, %1, %2;" : "+r"(v) : "r"(one), "r"(K2));
      } else if (MIX == 8) {             // 4 x popc
        asm("popc.b32 %0, %0;" : "+r"(v));
        asm("popc.b32 %0, %0;" : "+r"(v));
        asm("popc.b32 %0, %0;" : "+r"(v));
        asm("popc.b32 %0, %0;" : "+r"(v));
      } else if (MIX == 9) {             // 4 x shf (funnel)
        asm("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(v) : "r"(K2), "r"(K1));
        asm("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(v) : "r"(K1), "r"(K2));
        asm("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(v) : "r"(K2), "r"(K1));
      } else if (MIX == 10) {            // 4 x setp+selp (ISETP / SEL)
        uint32_t t;
        asm("{.reg .pred p; setp.lt.u32 p, %1, %2; selp.u32 %0, %1, %2, p;}" : "=r"(t) : "r"(v), "r"(K1)); v = t + 0;
        asm("{.reg .pred p; setp.lt.u32 p, %1, %2; selp.u32 %0, %1, %2, p;}" : "=r"(t) : "r"(v), "r"(K2)); v = t;
      } else if (MIX == 11) {            // 4 x bfind (FLO)
        asm("bfind.u32 %0, %0;" : "+r"(v));
        asm("bfind.u32 %0, %0;" : "+r"(v));
        asm("bfind.u32 %0, %0;" : "+r"(v));
        asm("bfind.u32 %0, %0;" : "+r"(v));
      }
      x[c] = v;
    }
  }
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < NCH; c++) acc ^= x[c];
  if (acc == 0x12345678u) out[0] = acc;
}

template <int MIX>
void run(const char* name, uint32_t* d, int sms) {
  const int iters = 4096, thr = 512, blocks = sms * 4;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k<MIX><<<blocks, thr>>>(d, 1, 1, 16);
  cudaEventRecord(a);
  k<MIX><<<blocks, thr>>>(d, 1, 1, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double warp_inst = (double)blocks * thr / 32 * iters * NCH * 4;
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-28s %.3f warp-inst/cycle/SMSP\n", name, warp_inst / cyc / sms / 4);
}

int main() {
  uint32_t* d; cudaMalloc(&d, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("4 lop3", d, sms); run<1>("4 add", d, sms); run<2>("4 imad", d, sms);
  run<3>("4 dp4a", d, sms); run<4>("2 lop3 + 2 add", d, sms); run<5>("2 lop3 + 2 imad", d, sms);
  run<6>("2 lop3 + 2 dp4a", d, sms); run<7>("2 add + 2 imad", d, sms); run<8>("4 popc", d, sms);
  run<9>("4 shf", d, sms); run<10>("2 (isetp+sel)", d, sms); run<11>("4 bfind", d, sms);
  return 0;
}
