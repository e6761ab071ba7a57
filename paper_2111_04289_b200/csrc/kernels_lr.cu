// Linear Road aggregate pass (LR2S, LR1S/LR1T): framing + validation + field decode +
// pane assignment + partial group-by aggregation, one pass over the 70 B records.
//
// PAPER.md: Table IV LR2S "AVG(speed) ... GROUPBY (highway, direction, segment)",
// LR1 window self-join on vehicle; record size "70 B (per record, fixed)";
// operators Scan (CSV) / Projection / Aggregation (Table III).  Record grammar:
// DESIGN.md reading R1.
//
// Design (B200): persistent CTAs (one contiguous tile range each), 1-D bulk copies
// (cp.async.bulk, TMA engine) of 35,840 B tiles (512 records) into a 2-stage smem ring
// tracked by mbarriers; each thread decodes a record PAIR (140 B = 35 aligned words, so
// every word load is aligned and bank-conflict free: word stride 35 is odd), validates all
// 70 bytes per record with SWAR range checks, parses the decoded fields from registers.
// LR2: native u32 shared-memory atomics into a per-CTA table [2 pane slots][K keys]
// (K = 200 * num_xways); at the end (and every q.lr2_flush_tiles tiles, so that a u32 sum cannot
// wrap) the CTA adds its tables into the u64 pane accumulators, one RED.64 pair per key seen
// (no global atomics per record).  LMS_LR2_PARTIALS=1 (A/B only) keeps round 1's per-CTA
// partials merged by the close.  LR1 (k_lr1_agg below): warp-owned
// 64-record tiles, dictionary-mapped (or dense) vehicle counts per pane (global REDs) and the
// projection of a 16 B row into the retained FIFO at deterministic positions.
#include "common.cuh"

#include <mutex>

namespace lms {
namespace {

constexpr int kLrThreads = 256;
constexpr int kLrStages = 2;
constexpr int kPairWords = 35;

// ---- compile-time validation constants for a record pair ---------------------------
__host__ __device__ constexpr bool lr_is_comma(int r) {
  return r == 1 || r == 8 || r == 19 || r == 23 || r == 27 || r == 29 || r == 31 || r == 35 ||
         r == 44 || r == 53 || r == 56 || r == 59 || r == 61 || r == 66;
}
__host__ __device__ constexpr uint32_t lr_expect_byte(int b) {
  return (b % 70) == 69 ? 0x0Au : (lr_is_comma(b % 70) ? 0x2Cu : 0x30u);
}
__host__ __device__ constexpr uint32_t lr_bias_byte(int b) {
  // byte ok iff (x = byte ^ expect) <= limit; bias = 0x7F - limit
  return ((b % 70) == 69 || lr_is_comma(b % 70)) ? 0x7Fu : 0x76u;
}
__host__ __device__ constexpr uint32_t lr_word(int j, bool bias) {
  uint32_t v = 0;
  for (int k = 0; k < 4; k++) v |= (bias ? lr_bias_byte(4 * j + k) : lr_expect_byte(4 * j + k)) << (8 * k);
  return v;
}

// Field decode, SWAR on digit bytes at compile-time offsets of the pair words.  Only records
// that lr_validate_pair accepted are used, so every field byte is an ASCII digit here.
// bytes4<B>: bytes [B, B+4) of the pair, first byte in the low byte.
template <int B>
__device__ __forceinline__ uint32_t bytes4(const uint32_t (&w)[kPairWords]) {
  if constexpr ((B & 3) == 0) return w[B >> 2];
  else return __funnelshift_r(w[B >> 2], w[(B >> 2) + 1], (B & 3) * 8);
}
// value of 4 digit values (first = most significant): pairs 10*d0+d1, 10*d2+d3 land in bytes 1
// and 3 of d * 0xA01 (each <= 99: no carries), PRMT moves them to bytes 0 and 2, and
// (p * (100 << 16 | 1)) >> 16 = 100 * pair0 + pair1 (the same identity as kernels_cm.cu swar4d,
// checked in tests/test_kernel_math.py)
__device__ __forceinline__ uint32_t lr_swar4d(uint32_t d) {
  const uint32_t p = __byte_perm(d * 0xA01u, 0u, 0x4341u);
  return (p * 0x640001u) >> 16;
}
// N <= 4 digits at byte B: the digit values of the field's bytes shifted to the top of the word
// (zero digits come in below).  Subtracting '0' cannot disturb the field's bytes: a borrow only
// runs from a non-digit byte toward later (higher) bytes, and the field's bytes come first.
template <int B, int N>
__device__ __forceinline__ uint32_t dec_u32(const uint32_t (&w)[kPairWords]) {
  static_assert(N >= 1 && N <= 4, "1..4 digits");
  const uint32_t d = bytes4<B>(w) - 0x30303030u;
  if constexpr (N == 1) return d & 0xFFu;
  else return lr_swar4d(d << (8 * (4 - N)));
}
template <int B>
__device__ __forceinline__ uint32_t dec_u32_6(const uint32_t (&w)[kPairWords]) {   // 6 digits
  return dec_u32<B, 4>(w) * 100u + dec_u32<B + 4, 2>(w);
}
template <int B>
__device__ __forceinline__ unsigned long long dec_u64_10(const uint32_t (&w)[kPairWords]) {   // 10 digits
  const uint32_t hi8 = dec_u32<B, 4>(w) * 10000u + dec_u32<B + 4, 4>(w);
  return (unsigned long long)hi8 * 100ull + dec_u32<B + 8, 2>(w);
}

struct LrRec {
  uint32_t ts, speed, xway, lane, dir, seg;
  unsigned long long vid;
};

template <int BASE, bool NEED_VID>
__device__ __forceinline__ LrRec lr_decode(const uint32_t (&w)[kPairWords]) {
  LrRec r;
  r.ts = dec_u32_6<BASE + 2>(w);
  r.speed = dec_u32<BASE + 20, 3>(w);
  r.xway = dec_u32<BASE + 24, 3>(w);
  r.lane = dec_u32<BASE + 28, 1>(w);
  r.dir = dec_u32<BASE + 30, 1>(w);
  r.seg = dec_u32<BASE + 32, 3>(w);
  r.vid = NEED_VID ? dec_u64_10<BASE + 9>(w) : 0ull;
  return r;
}

// Validate both records of a pair; returns bit0 = A ok, bit1 = B ok.
__device__ __forceinline__ uint32_t lr_validate_pair(const uint32_t (&w)[kPairWords]) {
  uint32_t badA = 0, badB = 0;
#pragma unroll
  for (int j = 0; j < kPairWords; j++) {
    const uint32_t x = w[j] ^ lr_word(j, false);
    const uint32_t t = ((x & 0x7F7F7F7Fu) + lr_word(j, true)) | x;
    if (j < 17) badA |= t;
    else if (j == 17) { badA |= t & 0x0000FFFFu; badB |= t & 0xFFFF0000u; }
    else badB |= t;
  }
  return ((badA & 0x80808080u) == 0 ? 1u : 0u) | ((badB & 0x80808080u) == 0 ? 2u : 0u);
}

struct LrArgs {
  QueryDev q;
  SegTable segs;
  unsigned long long total_tiles;
};

// Issue the bulk copy for global tile `tile` into stage buffer `dst` (the <16 B remainder of
// a segment's last tile is copied by threads later).
template <bool EVICT_FIRST>
__device__ __forceinline__ void lr_issue(const SegTable& segs, SegCursor& c, unsigned long long tile,
                                        uint8_t* dst, uint64_t* bar) {
  c.seek(segs, tile);
  const unsigned long long off = (tile - c.base) * (unsigned long long)kLrTileBytes;
  const unsigned long long rem = segs.s[c.si].nbytes - off;
  const uint32_t bytes = (uint32_t)(rem < (unsigned long long)kLrTileBytes ? rem : kLrTileBytes);
  const uint32_t bulk = bytes & ~15u;
  mbar_arrive_expect_tx(bar, bulk);
  if (bulk) {
    if (EVICT_FIRST) bulk_g2s_evict_first(dst, segs.s[c.si].ptr + off, bulk, bar);
    else bulk_g2s(dst, segs.s[c.si].ptr + off, bulk, bar);
  }
}

// Add the CTA's [2 panes][K] u32 tables into the u64 pane accumulators (one RED.64 pair per
// key seen) and, if `zero`, clear them for further records.
__device__ __forceinline__ void lr2_add_tables(const QueryDev& q, const unsigned long long* slot_tag, uint32_t* tsum,
                                               uint32_t* tcnt, uint32_t K, int tid, bool zero) {
  for (int sl = 0; sl < 2; sl++) {
    const unsigned long long tg = slot_tag[sl];
    if (tg == kEmpty64 || (uint32_t)(tg >> 32) == kFail32) continue;
    const size_t gbase = (size_t)(uint32_t)(tg >> 32) * K;
    for (uint32_t k = tid; k < K; k += blockDim.x) {
      const uint32_t cv = tcnt[sl * K + k];
      if (cv) {
        atomicAdd(&q.acc_sum[gbase + k], (unsigned long long)tsum[sl * K + k]);
        atomicAdd(&q.acc_cnt[gbase + k], (unsigned long long)cv);
        if (zero) { tsum[sl * K + k] = 0; tcnt[sl * K + k] = 0; }
      }
    }
  }
}
template <int KIND>
__global__ void __launch_bounds__(kLrThreads, 2) k_lr_agg(const LrArgs a) {
  static_assert(KIND == kLR2S, "LR1 runs k_lr1_agg");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kLrStages];
  __shared__ unsigned long long slot_tag[2], loaded_tag[2];
  const QueryDev& q = a.q;
  uint8_t* stage = smem;
  uint32_t* tsum = reinterpret_cast<uint32_t*>(smem + kLrStages * kLrTileBytes);   // [2][K]
  uint32_t* tcnt = tsum + 2 * q.K;                                                  // [2][K]
  const uint32_t K = q.K;
  const int tid = threadIdx.x;

  // contiguous tile range of this CTA
  const unsigned long long T = a.total_tiles, G = gridDim.x;
  const unsigned long long t0 = T * blockIdx.x / G, t1 = T * (blockIdx.x + 1) / G;

  for (uint32_t i = tid; i < 4 * K; i += blockDim.x) tsum[i] = 0;
  if (tid < 2) slot_tag[tid] = loaded_tag[tid] = q.part_tag[blockIdx.x * 2 + tid];
  if (tid == 0) {
    for (int s = 0; s < kLrStages; s++) mbar_init(&full[s], 1);
    mbar_fence_init();
  }
  __syncthreads();
  SegCursor cur, iss;                          // consumer / producer cursors
  cur.init(a.segs);
  iss.init(a.segs);
  if (tid == 0) {
    for (int s = 0; s < kLrStages; s++)
      if (t0 + s < t1) lr_issue<false>(a.segs, iss, t0 + s, stage + s * kLrTileBytes, &full[s]);
  }

  const unsigned long long wm_prev = q.state->wm_prev;
  CtaCounters cnt{0, 0, 0, 0, kEmpty32, 0};
  uint32_t c_pane = kEmpty32, c_slot = 0, c_gslot = kFail32;   // cached slots of the last pane seen
  uint32_t tiles_since_flush = 0;

  for (unsigned long long t = t0; t < t1; t++) {
    const int s = (int)((t - t0) % kLrStages);
    const uint32_t ph = (uint32_t)(((t - t0) / kLrStages) & 1);
    cur.seek(a.segs, t);
    const int si = cur.si;
    const unsigned long long off = (t - cur.base) * (unsigned long long)kLrTileBytes;
    const unsigned long long rem = a.segs.s[si].nbytes - off;
    const uint32_t bytes = (uint32_t)(rem < (unsigned long long)kLrTileBytes ? rem : kLrTileBytes);
    const uint32_t nrec = bytes / kLrRecBytes;
    uint8_t* buf = stage + s * kLrTileBytes;
    mbar_wait(&full[s], ph);
    if (bytes & 15u) {   // segment tail: copy the last < 16 bytes by hand (uniform branch)
      const uint32_t bulk = bytes & ~15u;
      if ((uint32_t)tid < bytes - bulk) buf[bulk + tid] = a.segs.s[si].ptr[off + bulk + tid];
      __syncthreads();
    }

    const uint32_t pair = tid;
    const uint32_t recA = 2 * pair;
    if (recA < nrec) {
      uint32_t w[kPairWords];
      const uint32_t* wp = reinterpret_cast<const uint32_t*>(buf) + pair * kPairWords;
#pragma unroll
      for (int j = 0; j < kPairWords; j++) w[j] = wp[j];
      uint32_t ok = lr_validate_pair(w);
      if (recA + 1 >= nrec) ok &= 1u;   // odd tail: record B does not exist
      LrRec rr[2] = {lr_decode<0, false>(w), lr_decode<70, false>(w)};
#pragma unroll
      for (int h = 0; h < 2; h++) {
        if (recA + h >= nrec) break;
        cnt.n++;
        const LrRec& r = rr[h];
        // Linear Road domains (reading R1): Dir in {0,1}, Seg <= 99, XWay < num_xways
        const bool valid = ((ok >> h) & 1u) && r.dir <= 1u && r.seg <= 99u && r.xway < q.num_xways;
        if (!valid) { cnt.bad++; continue; }
        if (wm_prev != 0 && (unsigned long long)r.ts + 1ull < wm_prev) { cnt.late++; continue; }   // R7
        cnt.ts_min = min(cnt.ts_min, r.ts);
        cnt.ts_max1 = max(cnt.ts_max1, r.ts + 1u);
        const uint32_t p = pane_of(r.ts, q.S, q.div_magic);
        const uint32_t key = (r.xway * 2u + r.dir) * 100u + r.seg;
        if (p != c_pane) {   // find / claim a local pane slot (tag = acc slot << 32 | pane)
          c_pane = p;
          local_slot(slot_tag, q, p, c_slot, c_gslot);
        }
        if (c_gslot == kFail32) { cnt.overflow++; continue; }
        if (c_slot < 2) {
          atomicAdd(&tsum[c_slot * K + key], r.speed);
          atomicAdd(&tcnt[c_slot * K + key], 1u);
        } else {
          const size_t g = (size_t)c_gslot * K + key;
          atomicAdd(&q.acc_sum[g], (unsigned long long)r.speed);
          atomicAdd(&q.acc_cnt[g], 1ull);
        }
      }
    }
    __syncthreads();   // stage s fully consumed
    if (tid == 0 && t + kLrStages < t1) lr_issue<false>(a.segs, iss, t + kLrStages, buf, &full[s]);
    // bound the u32 tables (CTA-uniform): q.lr2_flush_tiles (<= 8192) tiles of 512 records at
    // speed <= 999 stay below 2^32
    if (++tiles_since_flush == q.lr2_flush_tiles && t + 1 < t1) {
      lr2_add_tables(q, slot_tag, tsum, tcnt, K, tid, true);
      tiles_since_flush = 0;
      __syncthreads();
    }
  }

  if (q.lr2_direct) {
    // add this CTA's tables into the pane accumulators (one RED.64 pair per key seen): the
    // close then has nothing to merge, and a batch that closes no instance skips it entirely
    __syncthreads();
    lr2_add_tables(q, slot_tag, tsum, tcnt, K, tid, false);
  } else {
    __syncthreads();
    // write this CTA's pane partials: overwrite on the batch's first launch (the tag was
    // empty when loaded), accumulate when an earlier launch of the same batch wrote the slot
    uint32_t* part = q.part32 + (size_t)blockIdx.x * 4 * K;
    for (int sl = 0; sl < 2; sl++) {
      const unsigned long long tg = slot_tag[sl];
      if (tg == kEmpty64 || (uint32_t)(tg >> 32) == kFail32) continue;
      const bool fresh = loaded_tag[sl] == kEmpty64;
      for (uint32_t k = tid; k < K; k += blockDim.x) {
        const uint32_t sv = tsum[sl * K + k], cv = tcnt[sl * K + k];
        if (fresh) {
          part[(sl * 2 + 0) * K + k] = sv;
          part[(sl * 2 + 1) * K + k] = cv;
        } else if (cv) {
          part[(sl * 2 + 0) * K + k] += sv;
          part[(sl * 2 + 1) * K + k] += cv;
        }
      }
    }
    if (tid < 2) {
      const unsigned long long tg = slot_tag[tid];
      q.part_tag[blockIdx.x * 2 + tid] = ((uint32_t)(tg >> 32) == kFail32) ? kEmpty64 : tg;
    }
  }
  flush_counters(cnt, q.state);
}

// ---------------------------------------------------------------------------------------
// LR1 (LR1S / LR1T) aggregate pass: warp-owned tiles, no CTA barrier in the loop.
//
// Every warp walks its own contiguous range of 64-record warp tiles (4480 B, one bulk copy
// each) through a 2-stage smem ring; lane l decodes records 2l, 2l+1 of the tile (the 35-word
// pair layout of k_lr_agg: word stride 35 is odd, so the pair loads are bank-conflict free).
// Per record: validation, pane, vehicle index (dictionary: both records' first probes issued
// together, dict_get2; dense ids: the id itself), one RED.32 into the pane's vehicle counts,
// and its 16 B projected row into the retained FIFO.  FIFO positions are deterministic: the
// FIFO's count at launch start (read by every CTA before any CTA finishes) + tile * 64 + record
// (tail positions of a segment's last tile are written as holes), and the launch's last CTA
// advances the count by tiles * 64 — no per-tile reservation atomic and no CTA barrier.
constexpr int kLr1Warps = 4;
constexpr int kLr1Threads = kLr1Warps * 32;
constexpr int kLr1CtasPerSm = 5;
constexpr int kLr1TileRecs = 64;
constexpr int kLr1TileBytes = kLr1TileRecs * kLrRecBytes;   // 4480 = 16 * 280
constexpr int kLr1Stages = 2;

struct Lr1Args {
  QueryDev q;
  SegTable segs;
  unsigned long long total_tiles;
};

// Producer side of a warp's tile walk: segment / tile within it.
struct Lr1Iter {
  int si;
  unsigned long long t, seg_end;     // global tile index; first tile of the next segment
  __device__ __forceinline__ void init(const SegTable& s, unsigned long long tile) {
    si = 0;
    while (si + 1 < s.n && tile >= s.tile_prefix[si + 1]) si++;
    t = tile;
    seg_end = s.tile_prefix[si + 1];
  }
  __device__ __forceinline__ void next(const SegTable& s) {
    t++;
    while (t >= seg_end && si + 1 < s.n) { si++; seg_end = s.tile_prefix[si + 1]; }
  }
};

// Issue tile `it` into stage `dst` (shared-window address); returns its byte count (the < 16 B
// remainder of a segment's last tile is copied by lane 0 here: the stage is free).
__device__ __forceinline__ uint32_t lr1_issue(const SegTable& s, const Lr1Iter& it, uint32_t dst, uint32_t bar,
                                              int lane) {
  const unsigned long long off = (it.t - s.tile_prefix[it.si]) * (unsigned long long)kLr1TileBytes;
  const unsigned long long rem = s.s[it.si].nbytes - off;
  const uint32_t bytes = (uint32_t)(rem < (unsigned long long)kLr1TileBytes ? rem : kLr1TileBytes);
  const uint32_t bulk = bytes & ~15u;
  if (lane == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bulk) : "memory");
    const uint8_t* src = s.s[it.si].ptr + off;
    // read-once input: L2 evict-first, so the 700 MB stream does not push the vehicle
    // dictionary and the live panes' counts out of L2
    if (bulk)
      asm volatile("{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
                   " cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}"
                   ::"r"(dst), "l"(src), "r"(bulk), "r"(bar) : "memory");
    for (uint32_t i = bulk; i < bytes; i++)
      asm volatile("st.shared.u8 [%0], %1;" ::"r"(dst + i), "r"((uint32_t)src[i]));
  }
  return bytes;
}

__global__ void __launch_bounds__(kLr1Threads, kLr1CtasPerSm) k_lr1_agg(const Lr1Args a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kLr1Warps][kLr1Stages];
  const QueryDev& q = a.q;
  DevState* st = q.state;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned long long T = a.total_tiles, GW = (unsigned long long)gridDim.x * kLr1Warps;
  const unsigned long long gw = (unsigned long long)blockIdx.x * kLr1Warps + warp;
  const unsigned long long t0 = T * gw / GW, t1 = T * (gw + 1) / GW;
  const uint32_t K = q.K;
  // the FIFO count is only advanced by this launch's last CTA, after every CTA read it here
  const uint32_t fcur = *(volatile uint32_t*)&st->fifo_cur;
  const unsigned long long fbase = *(volatile unsigned int*)&st->fifo_count[fcur];
  Lr1Retained* const fifo = q.fifo[fcur];
  const unsigned long long wm_prev = st->wm_prev;
  if (lane == 0) {
    for (int s = 0; s < kLr1Stages; s++) mbar_init(&full[warp][s], 1);
    mbar_fence_init();
  }
  __syncwarp();
  const uint32_t stage_s = smem_addr(smem + warp * (kLr1Stages * kLr1TileBytes));
  const uint32_t full_s = smem_addr(&full[warp][0]);
  const uint32_t ntiles = (uint32_t)(t1 - t0);
  Lr1Iter iss;
  iss.init(a.segs, t0);
  uint32_t bytes0 = 0, bytes1 = 0;             // bytes of the tiles in stages 0 / 1
  unsigned long long tile0 = 0, tile1 = 0;     // their global tile indices
  if (ntiles > 0) { tile0 = iss.t; bytes0 = lr1_issue(a.segs, iss, stage_s, full_s, lane); iss.next(a.segs); }
  if (ntiles > 1) { tile1 = iss.t; bytes1 = lr1_issue(a.segs, iss, stage_s + kLr1TileBytes, full_s + 8u, lane); iss.next(a.segs); }

  CtaCounters cnt{0, 0, 0, 0, kEmpty32, 0};
  uint32_t c_pane = kEmpty32, c_gslot = kFail32;   // cached slot of the last pane seen
  for (uint32_t it = 0; it < ntiles; it++) {
    const uint32_t s = it & 1u;
    const uint32_t bytes = s ? bytes1 : bytes0;
    const unsigned long long tile = s ? tile1 : tile0;
    const uint32_t sb = stage_s + s * (uint32_t)kLr1TileBytes;
    mbar_wait_shared(full_s + 8u * s, (it >> 1) & 1u);
    __syncwarp();                                // (lane 0's remainder bytes, tail tiles)
    const uint32_t nrec = bytes / kLrRecBytes;
    const uint32_t recA = 2u * lane;
    LrRec rr[2];
    uint32_t ok = 0;
    if (recA < nrec) {
      uint32_t w[kPairWords];
#pragma unroll
      for (int j = 0; j < kPairWords; j++) w[j] = lds_u32(sb + 4u * (lane * kPairWords + j));
      ok = lr_validate_pair(w);
      if (recA + 1 >= nrec) ok &= 1u;          // odd tail: record B does not exist
      rr[0] = lr_decode<0, true>(w);
      rr[1] = lr_decode<70, true>(w);
    }
    bool use[2] = {false, false};
    uint32_t gslot[2] = {kFail32, kFail32};
#pragma unroll
    for (int h = 0; h < 2; h++) {
      if (recA + h >= nrec) continue;
      cnt.n++;
      const LrRec& r = rr[h];
      // Linear Road domains (reading R1): Dir in {0,1}, Seg <= 99, XWay < num_xways
      const bool valid = ((ok >> h) & 1u) && r.dir <= 1u && r.seg <= 99u && r.xway < q.num_xways;
      if (!valid) cnt.bad++;
      else if (wm_prev != 0 && (unsigned long long)r.ts + 1ull < wm_prev) cnt.late++;   // R7
      else {
        cnt.ts_min = min(cnt.ts_min, r.ts);
        cnt.ts_max1 = max(cnt.ts_max1, r.ts + 1u);
        const uint32_t p = pane_of(r.ts, q.S, q.div_magic);
        if (p != c_pane) { c_pane = p; c_gslot = claim_slot(q, p); }
        gslot[h] = c_gslot;
        use[h] = c_gslot != kFail32;
        if (!use[h]) cnt.overflow++;
      }
    }
    uint32_t vidx[2];
    if (q.lr1_dense) {
      // lr1_dense (multi-GPU, LMS_FLAG_DENSE_VEHICLES): the vehicle id is the index; a VID >=
      // max_keys rejects the batch (LMS_EINVAL at its completion), never silent overflow
#pragma unroll
      for (int h = 0; h < 2; h++) {
        vidx[h] = use[h] && rr[h].vid < K ? (uint32_t)rr[h].vid : kEmpty32;
        if (use[h] && rr[h].vid >= K) atomicExch(&st->vid_range, 1u);
      }
    } else {
      dict_get2(q.dict, rr[0].vid, use[0], rr[1].vid, use[1], st, vidx[0], vidx[1]);
    }
    const unsigned long long pos0 = fbase + tile * (unsigned long long)kLr1TileRecs + recA;
#pragma unroll
    for (int h = 0; h < 2; h++) {
      if (use[h]) {
        if (vidx[h] == kEmpty32) cnt.overflow++;
        else atomicAdd(&q.acc_cnt32[(size_t)gslot[h] * K + vidx[h]], 1u);
      }
      // projected row (a hole, vidx = kEmpty32, for a dropped record or a tail position)
      Lr1Retained row;
      const bool live = recA + h < nrec;
      const LrRec& r = rr[h];
      row.ts = live ? r.ts : 0u;
      row.vidx = use[h] ? vidx[h] : kEmpty32;
      row.speed = live ? (uint16_t)r.speed : 0; row.xway = live ? (uint16_t)r.xway : 0;
      row.seg = live ? (uint16_t)r.seg : 0; row.lane = live ? (uint8_t)r.lane : 0; row.dir = live ? (uint8_t)r.dir : 0;
      if (pos0 + h < q.fifo_cap) {
        __stcs(reinterpret_cast<uint4*>(fifo + pos0 + h), *reinterpret_cast<const uint4*>(&row));
      } else if (use[h] && vidx[h] != kEmpty32) {
        atomicExch(&st->fifo_overflow, 1u);
        cnt.overflow++;
      }
    }
    __syncwarp();                                // stage s consumed by every lane
    if (it + kLr1Stages < ntiles) {
      const unsigned long long tn = iss.t;
      const uint32_t b2 = lr1_issue(a.segs, iss, sb, full_s + 8u * s, lane);
      iss.next(a.segs);
      bytes0 = s ? bytes0 : b2;
      bytes1 = s ? b2 : bytes1;
      tile0 = s ? tile0 : tn;
      tile1 = s ? tn : tile1;
    }
  }
  flush_counters(cnt, st, smem);                 // (syncs the CTA: the stages are free)
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&st->lr1_ticket, 1u) == gridDim.x - 1) {   // last CTA of the launch
      st->fifo_count[fcur] = (unsigned int)min(fbase + T * (unsigned long long)kLr1TileRecs, 0xFFFFFFFFull);
      st->lr1_ticket = 0;
      __threadfence();
    }
  }
}

}  // namespace

// Load every kernel of this file now (CUDA 12 loads kernels lazily, at first launch, and a
// lazy load waits for the device: a first launch behind a running spin-wait kernel of another
// handle — the multi-GPU device barriers on a shared GPU — would wait for that spin to time
// out).  Called once per process from lms_query_create.
void preload_lr_kernels() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_lr_agg<kLR2S>);
  cudaFuncGetAttributes(&fa, k_lr1_agg);
}

int lr_agg_ctas(const QueryDev& q) {
  static int nsm = -1;
  if (nsm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return (q.kind == kLR1S || q.kind == kLR1T) ? nsm * kLr1CtasPerSm : nsm * 2;
}

uint64_t lr_tiles(const QueryDev& q, uint64_t nbytes) {
  const uint64_t recs = nbytes / kLrRecBytes, per = (q.kind == kLR1S || q.kind == kLR1T) ? kLr1TileRecs : kLrTileRecs;
  return (recs + per - 1) / per;
}

size_t lr_agg_smem(const QueryDev& q) {
  const bool lr1 = (q.kind == kLR1S || q.kind == kLR1T);
  return lr1 ? (size_t)kLr1Warps * kLr1Stages * kLr1TileBytes
             : (size_t)kLrStages * kLrTileBytes + (size_t)4 * q.K * sizeof(uint32_t);
}

// cudaFuncSetAttribute once per (kernel, device, size): it is not a per-launch call (and the
// driver may serialise it against running work, which the multi-GPU device-side barriers of
// other handles on the same device must never wait behind).
static cudaError_t set_smem_once(const void* fn, int bytes) {
  static std::mutex mu;
  static const void* done_fn[16];
  static int done_dev[16], done_bytes[16], n_done = 0;
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  cudaGetDevice(&dev);
  for (int i = 0; i < n_done; i++)
    if (done_fn[i] == fn && done_dev[i] == dev && done_bytes[i] >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess && n_done < 16) { done_fn[n_done] = fn; done_dev[n_done] = dev; done_bytes[n_done] = bytes; n_done++; }
  return e;
}

cudaError_t launch_lr_agg(const QueryDev& q, const SegTable& segs, cudaStream_t st) {
  LrArgs a;
  a.q = q;
  a.segs = segs;
  a.total_tiles = segs.tile_prefix[segs.n];
  if (a.total_tiles == 0) return cudaSuccess;
  const size_t smem = lr_agg_smem(q);
  const int grid = (int)q.n_agg_ctas;
  cudaError_t e;
  switch (q.kind) {
    case kLR2S:
      e = set_smem_once((const void*)k_lr_agg<kLR2S>, (int)smem);
      if (e != cudaSuccess) return e;
      k_lr_agg<kLR2S><<<grid, kLrThreads, smem, st>>>(a);
      break;
    case kLR1S:
    case kLR1T: {
      e = set_smem_once((const void*)k_lr1_agg, (int)smem);
      if (e != cudaSuccess) return e;
      Lr1Args b;
      b.q = q;
      b.segs = segs;
      b.total_tiles = a.total_tiles;
      k_lr1_agg<<<grid, kLr1Threads, smem, st>>>(b);
      break;
    }
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace lms
