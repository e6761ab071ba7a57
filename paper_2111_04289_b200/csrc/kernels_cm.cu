// Cluster Monitoring aggregate pass (CM1S/CM1T, CM2S): newline framing + field decode +
// validation + predicate + warp-ballot compaction + pane partial aggregation.
//
// PAPER.md: Table IV CM1 "SUM(cpu) ... GROUPBY category ORDERBY SUM(cpu)", CM2
// "AVG(cpu) ... WHERE (eventType == 1) GROUPBY jobId"; record size "130 ~ 145 B (per record,
// variable)"; operators Scan (CSV) / Filtering / Projection / Aggregation (Table III).
// Record grammar: DESIGN.md reading R1 (13-column task_events line, <= 255 B + '\n').
//
// Design (B200): persistent CTAs over contiguous 32 KB tiles; each tile is bulk-copied (TMA
// engine, cp.async.bulk) into a 3-stage smem ring together with a 16 B left halo (to see the
// byte before the tile) and a 256 B right halo (to finish the last record that STARTS in the
// tile: a record belongs to the tile holding its first byte).  Thread j owns the 128 B chunk
// j: it builds the chunk's newline bitmask with SWAR zero-byte tests, derives record starts
// (byte after '\n'), then walks each of its records word by word to locate the 12 commas
// and the terminating '\n' (SWAR again), validates and decodes ts, jobId, eventType,
// category, cpu (fixed-point cpu*1e6).  CM2: survivors of eventType == 1 are compacted with
// warp ballots into a dense smem list, then processed by full warps (dictionary jobId ->
// index, two RED.64 into the pane accumulators).  CM1: per-warp ballot/REDUX reduction per
// (pane, category), per-warp smem accumulators, one RED.64 pair per CTA and key at the end.
#include "common.cuh"

namespace lms {
namespace {

constexpr int kCmThreads = 256;
constexpr int kCmStages = 3;
constexpr int kChunk = kCmTile / kCmThreads;   // 128 B per thread
static_assert(kChunk == 128, "chunk");

__device__ __forceinline__ uint32_t zero_bytes(uint32_t y) {
  // bit 7 of each byte set iff that byte of y is zero (exact, no borrow artefacts)
  const uint32_t t = (y & 0x7F7F7F7Fu) + 0x7F7F7F7Fu;
  return ~(t | y | 0x7F7F7F7Fu);
}
__device__ __forceinline__ uint32_t nibble(uint32_t flags) {
  // compress bits 7,15,23,31 into bits 0..3
  return ((flags >> 7) * 0x00204081u) >> 21 & 0xFu;
}

struct CmArgs {
  QueryDev q;
  SegTable segs;
  unsigned long long total_tiles;
};

__device__ __forceinline__ void seg_of_tile(const SegTable& s, unsigned long long tile, int& si,
                                            unsigned long long& local) {
  si = 0;
  while (si + 1 < s.n && tile >= s.tile_prefix[si + 1]) si++;
  local = tile - s.tile_prefix[si];
}

struct TileGeom {
  const uint8_t* seg;
  unsigned long long seg_len, off;   // tile starts at seg + off
  uint32_t lo, hi;                   // valid smem bytes [lo, hi) (relative to stage start)
  uint32_t payload;                  // tile payload bytes (<= kCmTile)
};

__device__ __forceinline__ TileGeom cm_geom(const SegTable& segs, unsigned long long tile) {
  int si;
  unsigned long long lt;
  seg_of_tile(segs, tile, si, lt);
  TileGeom g;
  g.seg = segs.s[si].ptr;
  g.seg_len = segs.s[si].nbytes;
  g.off = lt * (unsigned long long)kCmTile;
  const unsigned long long rem = g.seg_len - g.off;
  g.payload = (uint32_t)(rem < (unsigned long long)kCmTile ? rem : kCmTile);
  g.lo = lt == 0 ? kCmHaloL : 0;
  const unsigned long long end = (rem < (unsigned long long)(kCmTile + kCmHaloR)) ? rem : (kCmTile + kCmHaloR);
  g.hi = kCmHaloL + (uint32_t)end;
  return g;
}

__device__ __forceinline__ void cm_issue(const SegTable& segs, unsigned long long tile, uint8_t* dst,
                                         uint64_t* bar) {
  const TileGeom g = cm_geom(segs, tile);
  const uint32_t bulk = (g.hi - g.lo) & ~15u;
  mbar_arrive_expect_tx(bar, bulk);
  if (bulk) bulk_g2s(dst + g.lo, g.seg + g.off - kCmHaloL + g.lo, bulk, bar);
}

struct CmRec {
  uint32_t ts;
  unsigned long long job;
  uint32_t event, cat, cpu_m;
};

// Parse one line starting at smem offset s (stage-relative); limit = first invalid byte.
// Returns: 1 valid, 0 malformed.  *next = offset after the terminating '\n' (or limit).
__device__ __forceinline__ int cm_parse(const uint8_t* buf, uint32_t s, uint32_t limit, CmRec& r,
                                        uint32_t& end_out) {
  uint32_t c[13];
  uint32_t nc = 0;
  uint32_t e = 0xFFFFFFFFu;
  const uint32_t stop = min(limit, s + kCmMaxLine + 1);   // '\n' must be at <= s + 255
  uint32_t a = s & ~3u;
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(buf);
  while (a < stop) {
    const uint32_t w = wp[a >> 2];
    uint32_t nl = nibble(zero_bytes(w ^ 0x0A0A0A0Au));
    uint32_t cm = nibble(zero_bytes(w ^ 0x2C2C2C2Cu));
    // clip to [s, stop)
    uint32_t keep = 0xFu;
    if (a < s) keep &= (0xFu << (s - a)) & 0xFu;
    if (a + 4 > stop) keep &= (0xFu >> (a + 4 - stop));
    nl &= keep;
    cm &= keep;
    if (nl) {
      const uint32_t b = __ffs(nl) - 1;
      e = a + b;
      cm &= (1u << b) - 1u;
    }
    while (cm) {
      const uint32_t b = __ffs(cm) - 1;
      cm &= cm - 1;
      if (nc < 13) c[nc] = a + b;
      nc++;
    }
    if (e != 0xFFFFFFFFu) break;
    a += 4;
  }
  if (e == 0xFFFFFFFFu) {   // no '\n' within 256 bytes or before the segment end
    end_out = stop;
    return 0;
  }
  end_out = e + 1;
  if (nc != 12) return 0;
  // f0 ts: 1..9 digits in [s, c0)
  const uint32_t lts = c[0] - s;
  if (lts < 1 || lts > 9) return 0;
  uint32_t ts = 0;
  for (uint32_t i = s; i < c[0]; i++) {
    const uint32_t d = (uint32_t)buf[i] - 48u;
    if (d > 9u) return 0;
    ts = ts * 10u + d;
  }
  if (c[1] != c[0] + 1) return 0;   // f1 (missing info) empty
  const uint32_t lj = c[2] - c[1] - 1;
  if (lj < 1 || lj > 19) return 0;
  unsigned long long job = 0;
  for (uint32_t i = c[1] + 1; i < c[2]; i++) {
    const uint32_t d = (uint32_t)buf[i] - 48u;
    if (d > 9u) return 0;
    job = job * 10ull + d;
  }
  if (c[5] != c[4] + 2 || c[7] != c[6] + 2 || c[9] != c[8] + 9) return 0;
  const uint32_t ev = (uint32_t)buf[c[4] + 1] - 48u;
  const uint32_t cat = (uint32_t)buf[c[6] + 1] - 48u;
  if (ev > 9u || cat > 9u) return 0;
  const uint8_t* cp = buf + c[8] + 1;
  if (cp[1] != '.') return 0;
  uint32_t m = (uint32_t)cp[0] - 48u;
  if (m > 9u) return 0;
#pragma unroll
  for (int i = 2; i < 8; i++) {
    const uint32_t d = (uint32_t)cp[i] - 48u;
    if (d > 9u) return 0;
    m = m * 10u + d;
  }
  r.ts = ts;
  r.job = job;
  r.event = ev;
  r.cat = cat;
  r.cpu_m = m;
  return 1;
}

template <int KIND>
__global__ void __launch_bounds__(kCmThreads, 2) k_cm_agg(const CmArgs a) {
  constexpr bool kCM2 = (KIND == kCM2S);
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kCmStages];
  __shared__ unsigned long long slot_tag[2];
  // CM2 compaction list
  __shared__ unsigned long long l_job[kCmThreads];
  __shared__ uint32_t l_m[kCmThreads], l_p[kCmThreads];
  __shared__ uint32_t l_n;
  // CM1 per-warp accumulators [warp][slot][cat] (sum, count)
  __shared__ unsigned long long w_sum[kCmThreads / 32][2][10], w_cnt[kCmThreads / 32][2][10];

  const QueryDev& q = a.q;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long T = a.total_tiles, G = gridDim.x;
  const unsigned long long t0 = T * blockIdx.x / G, t1 = T * (blockIdx.x + 1) / G;

  if (!kCM2) {
    for (int i = tid; i < (kCmThreads / 32) * 20; i += blockDim.x) {
      (&w_sum[0][0][0])[i] = 0;
      (&w_cnt[0][0][0])[i] = 0;
    }
  }
  if (tid < 2) slot_tag[tid] = kEmpty64;
  if (tid == 0) {
    for (int s = 0; s < kCmStages; s++) mbar_init(&full[s], 1);
    mbar_fence_init();
    l_n = 0;
  }
  __syncthreads();
  if (tid == 0)
    for (int s = 0; s < kCmStages; s++)
      if (t0 + s < t1) cm_issue(a.segs, t0 + s, smem + s * kCmStage, &full[s]);

  const unsigned long long wm_prev = q.state->wm_prev;
  CtaCounters cnt{0, 0, 0, 0, kEmpty32, 0};
  uint32_t c_pane = kEmpty32, c_slot = 0, c_gslot = kFail32;   // cached slots of the last pane seen

  for (unsigned long long t = t0; t < t1; t++) {
    const int s = (int)((t - t0) % kCmStages);
    const uint32_t ph = (uint32_t)(((t - t0) / kCmStages) & 1);
    uint8_t* buf = smem + s * kCmStage;
    const TileGeom g = cm_geom(a.segs, t);
    mbar_wait(&full[s], ph);
    {   // remainder bytes the bulk copy could not move (segment tail, < 16 B)
      const uint32_t bulk_end = g.lo + ((g.hi - g.lo) & ~15u);
      if (bulk_end < g.hi) {
        if ((uint32_t)tid < g.hi - bulk_end) buf[bulk_end + tid] = g.seg[g.off - kCmHaloL + bulk_end + tid];
        __syncthreads();
      }
    }
    // ---- framing: starts of records in my chunk --------------------------------------
    const uint32_t c0 = kCmHaloL + tid * kChunk;                 // stage offset of my chunk
    const uint32_t cend = kCmHaloL + g.payload;                  // end of tile payload
    unsigned long long st_lo = 0, st_hi = 0;                     // start bits of bytes c0..c0+127
    if (c0 < cend) {
      const uint4* v = reinterpret_cast<const uint4*>(buf + c0);
      unsigned long long nlm[2] = {0, 0};
#pragma unroll
      for (int k = 0; k < 8; k++) {
        const uint4 x = v[k];
        const uint32_t n = nibble(zero_bytes(x.x ^ 0x0A0A0A0Au)) | (nibble(zero_bytes(x.y ^ 0x0A0A0A0Au)) << 4) |
                           (nibble(zero_bytes(x.z ^ 0x0A0A0A0Au)) << 8) | (nibble(zero_bytes(x.w ^ 0x0A0A0A0Au)) << 12);
        nlm[k >> 2] |= (unsigned long long)n << ((k & 3) * 16);
      }
      const bool carry = (c0 == kCmHaloL && g.lo == kCmHaloL) ? true : (buf[c0 - 1] == '\n');
      st_lo = (nlm[0] << 1) | (carry ? 1ull : 0ull);
      st_hi = (nlm[1] << 1) | (nlm[0] >> 63);
      const uint32_t nvalid = min(128u, cend - c0);               // starts only inside the payload
      if (nvalid < 128) {
        if (nvalid <= 64) { st_hi = 0; st_lo &= (nvalid == 64) ? ~0ull : ((1ull << nvalid) - 1); }
        else st_hi &= (1ull << (nvalid - 64)) - 1;
      }
    }
    // ---- parse my records (rounds: one record per thread per round) -------------------
    while (true) {
      int have = 0;
      CmRec r{0, 0, 0, 0, 0};
      bool surv = false;
      if (st_lo | st_hi) {
        uint32_t b;
        if (st_lo) { b = __ffsll(st_lo) - 1; st_lo &= st_lo - 1; }
        else { b = 64 + __ffsll(st_hi) - 1; st_hi &= st_hi - 1; }
        uint32_t endo;
        have = 1;
        cnt.n++;
        const int ok = cm_parse(buf, c0 + b, g.hi, r, endo);
        if (!ok) { cnt.bad++; have = 0; }
        else if (wm_prev != 0 && (unsigned long long)r.ts + 1ull < wm_prev) { cnt.late++; have = 0; }
        else {
          cnt.ts_min = min(cnt.ts_min, r.ts);
          cnt.ts_max1 = max(cnt.ts_max1, r.ts + 1u);
          surv = kCM2 ? (r.event == 1u) : true;                   // WHERE (eventType == 1)
        }
      }
      uint32_t p = surv ? pane_of(r.ts, q.S, q.div_magic) : 0;
      if (kCM2) {
        // warp-ballot compaction of survivors into the dense CTA list
        const uint32_t bal = __ballot_sync(0xffffffffu, surv);
        uint32_t base = 0;
        if (lane == 0 && bal) base = atomicAdd(&l_n, __popc(bal));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (surv) {
          const uint32_t pos = base + __popc(bal & ((1u << lane) - 1u));
          l_job[pos] = r.job;
          l_m[pos] = r.cpu_m;
          l_p[pos] = p;
        }
        __syncthreads();
        const uint32_t n = l_n;
        for (uint32_t i = tid; i < n; i += blockDim.x) {          // full warps on survivors
          const uint32_t pp = l_p[i];
          if (pp != c_pane) { c_pane = pp; c_gslot = claim_slot(q, pp); }
          const uint32_t idx = c_gslot != kFail32 ? dict_get(q.dict, l_job[i], q.state) : kEmpty32;
          if (idx == kEmpty32) { cnt.overflow++; continue; }
          const size_t gi = (size_t)c_gslot * q.K + idx;
          atomicAdd(&q.acc_sum[gi], (unsigned long long)l_m[i]);
          atomicAdd(&q.acc_cnt[gi], 1ull);
        }
        __syncthreads();
        if (tid == 0) l_n = 0;
      } else {
        // CM1: reduce per (pane, category) inside the warp
        bool pend = surv;
        uint32_t left = __ballot_sync(0xffffffffu, pend);
        while (left) {
          const int leader = __ffs(left) - 1;
          const uint32_t lp = __shfl_sync(0xffffffffu, p, leader);
          const uint32_t lc = __shfl_sync(0xffffffffu, r.cat, leader);
          const bool me = pend && p == lp && r.cat == lc;
          const uint32_t mm = __ballot_sync(0xffffffffu, me);
          const uint32_t sm = __reduce_add_sync(0xffffffffu, me ? r.cpu_m : 0u);   // < 32 * 1e7
          if (lane == leader) {
            if (lp != c_pane) {
              c_pane = lp;
              local_slot(slot_tag, q, lp, c_slot, c_gslot);
            }
            if (c_gslot == kFail32) cnt.overflow += __popc(mm);
            else if (c_slot < 2) {
              w_sum[warp][c_slot][lc] += sm;
              w_cnt[warp][c_slot][lc] += __popc(mm);
            } else {
              const size_t gi = (size_t)c_gslot * q.K + lc;
              atomicAdd(&q.acc_sum[gi], (unsigned long long)sm);
              atomicAdd(&q.acc_cnt[gi], (unsigned long long)__popc(mm));
            }
          }
          if (me) pend = false;
          left &= ~mm;
          __syncwarp();   // order the leader's smem accumulator update before the next leader's
        }
      }
      if (!__syncthreads_or(st_lo | st_hi ? 1 : 0)) break;
    }
    __syncthreads();   // stage s consumed
    if (tid == 0 && t + kCmStages < t1) cm_issue(a.segs, t + kCmStages, buf, &full[s]);
  }

  if (!kCM2) {
    __syncthreads();
    if (tid < 20) {
      const int sl = tid / 10, c = tid % 10;
      const unsigned long long tg = slot_tag[sl];
      if (tg != kEmpty64 && (uint32_t)(tg >> 32) != kFail32) {
        unsigned long long sv = 0, cv = 0;
        for (int w = 0; w < kCmThreads / 32; w++) { sv += w_sum[w][sl][c]; cv += w_cnt[w][sl][c]; }
        if (cv) {
          const size_t gi = (size_t)(tg >> 32) * q.K + c;
          atomicAdd(&q.acc_sum[gi], sv);
          atomicAdd(&q.acc_cnt[gi], cv);
        }
      }
    }
  }
  flush_counters(cnt, q.state);
}

}  // namespace

int cm_agg_ctas(const QueryDev& q) {
  static int nsm = -1;
  if (nsm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  (void)q;
  return nsm * 2;
}

cudaError_t launch_cm_agg(const QueryDev& q, const SegTable& segs, cudaStream_t st) {
  CmArgs a;
  a.q = q;
  a.segs = segs;
  a.total_tiles = segs.tile_prefix[segs.n];
  if (a.total_tiles == 0) return cudaSuccess;
  const size_t smem = (size_t)kCmStages * kCmStage;
  const int grid = (int)q.n_agg_ctas;
  cudaError_t e;
  if (q.kind == kCM2S) {
    e = cudaFuncSetAttribute(k_cm_agg<kCM2S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_cm_agg<kCM2S><<<grid, kCmThreads, smem, st>>>(a);
  } else {
    e = cudaFuncSetAttribute(k_cm_agg<kCM1S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_cm_agg<kCM1S><<<grid, kCmThreads, smem, st>>>(a);
  }
  return cudaGetLastError();
}

}  // namespace lms
