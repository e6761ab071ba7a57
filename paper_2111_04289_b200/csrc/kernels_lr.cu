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
// (K = 200 * num_xways), written once per CTA to a partials array that the close kernel
// merges per key slice (no global atomics on the hot path).  LR1: dictionary-mapped
// vehicle counts per pane (global REDs) + projection of a 16 B row into the retained FIFO.
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

template <int B>
__device__ __forceinline__ uint32_t byte_at(const uint32_t (&w)[kPairWords]) {
  return (w[B >> 2] >> ((B & 3) * 8)) & 0xFFu;
}
template <int B, int N>
__device__ __forceinline__ uint32_t dec_u32(const uint32_t (&w)[kPairWords]) {
  uint32_t v = 0;
#pragma unroll
  for (int i = 0; i < N; i++) {
    // byte_at with a compile-time index after unrolling
    const int b = B + i;
    v = v * 10u + (((w[b >> 2] >> ((b & 3) * 8)) & 0xFFu) - 48u);
  }
  return v;
}
template <int B, int N>
__device__ __forceinline__ unsigned long long dec_u64(const uint32_t (&w)[kPairWords]) {
  unsigned long long v = 0;
#pragma unroll
  for (int i = 0; i < N; i++) {
    const int b = B + i;
    v = v * 10ull + (((w[b >> 2] >> ((b & 3) * 8)) & 0xFFu) - 48u);
  }
  return v;
}

struct LrRec {
  uint32_t ts, speed, xway, lane, dir, seg;
  unsigned long long vid;
};

template <int BASE, bool NEED_VID>
__device__ __forceinline__ LrRec lr_decode(const uint32_t (&w)[kPairWords]) {
  LrRec r;
  r.ts = dec_u32<BASE + 2, 6>(w);
  r.speed = dec_u32<BASE + 20, 3>(w);
  r.xway = dec_u32<BASE + 24, 3>(w);
  r.lane = dec_u32<BASE + 28, 1>(w);
  r.dir = dec_u32<BASE + 30, 1>(w);
  r.seg = dec_u32<BASE + 32, 3>(w);
  r.vid = NEED_VID ? dec_u64<BASE + 9, 10>(w) : 0ull;
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

template <int KIND>
__global__ void __launch_bounds__(kLrThreads, 2) k_lr_agg(const LrArgs a) {
  constexpr bool kLR1 = (KIND == kLR1S || KIND == kLR1T);
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kLrStages];
  __shared__ unsigned long long slot_tag[2], loaded_tag[2];
  __shared__ uint32_t s_fbase, s_fcur;      // LR1: this tile's reserved FIFO range
  const QueryDev& q = a.q;
  uint8_t* stage = smem;
  uint32_t* tsum = reinterpret_cast<uint32_t*>(smem + kLrStages * kLrTileBytes);   // [2][K]
  uint32_t* tcnt = tsum + 2 * q.K;                                                  // [2][K]
  const uint32_t K = q.K;
  const int tid = threadIdx.x;

  // contiguous tile range of this CTA
  const unsigned long long T = a.total_tiles, G = gridDim.x;
  const unsigned long long t0 = T * blockIdx.x / G, t1 = T * (blockIdx.x + 1) / G;

  if (!kLR1) {
    for (uint32_t i = tid; i < 4 * K; i += blockDim.x) tsum[i] = 0;
    if (tid < 2) slot_tag[tid] = loaded_tag[tid] = q.part_tag[blockIdx.x * 2 + tid];
  }
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
      if (t0 + s < t1) lr_issue<kLR1>(a.segs, iss, t0 + s, stage + s * kLrTileBytes, &full[s]);
  }

  const unsigned long long wm_prev = q.state->wm_prev;
  CtaCounters cnt{0, 0, 0, 0, kEmpty32, 0};
  uint32_t c_pane = kEmpty32, c_slot = 0, c_gslot = kFail32;   // cached slots of the last pane seen

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
    if (kLR1) {   // one FIFO reservation per tile (was one contended atomic per warp and record)
      if (tid == 0) {
        s_fcur = q.state->fifo_cur;
        s_fbase = atomicAdd(&q.state->fifo_count[s_fcur], nrec);
      }
    }
    mbar_wait(&full[s], ph);
    if (kLR1) __syncthreads();
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
      LrRec rr[2] = {lr_decode<0, kLR1>(w), lr_decode<70, kLR1>(w)};
#pragma unroll
      for (int h = 0; h < 2; h++) {
        if (recA + h >= nrec) break;
        cnt.n++;
        const LrRec& r = rr[h];
        // Linear Road domains (reading R1): Dir in {0,1}, Seg <= 99, XWay < num_xways
        const bool valid = ((ok >> h) & 1u) && r.dir <= 1u && r.seg <= 99u && r.xway < q.num_xways;
        if (kLR1) {
          // LR1: vehicle count of the record's pane + its projected row in the retained FIFO
          // at the tile's reserved position (a hole, vidx = kEmpty32, for a dropped record)
          uint32_t vidx = kEmpty32;
          if (!valid) cnt.bad++;
          else if (wm_prev != 0 && (unsigned long long)r.ts + 1ull < wm_prev) cnt.late++;   // R7
          else {
            cnt.ts_min = min(cnt.ts_min, r.ts);
            cnt.ts_max1 = max(cnt.ts_max1, r.ts + 1u);
            const uint32_t p = pane_of(r.ts, q.S, q.div_magic);
            if (p != c_pane) { c_pane = p; c_gslot = claim_slot(q, p); }
            // lr1_dense (multi-GPU, LMS_FLAG_DENSE_VEHICLES): the vehicle id is the index
            vidx = c_gslot == kFail32 ? kEmpty32
                 : q.lr1_dense ? (r.vid < K ? (uint32_t)r.vid : kEmpty32)
                               : dict_get(q.dict, r.vid, q.state);
            // dense-vehicle mode cannot represent a VID >= max_keys: the batch is rejected
            // (LMS_EINVAL at its completion), not silently counted as overflow
            if (q.lr1_dense && r.vid >= K && c_gslot != kFail32) atomicExch(&q.state->vid_range, 1u);
            if (vidx == kEmpty32) cnt.overflow++;
            else atomicAdd(&q.acc_cnt32[(size_t)c_gslot * K + vidx], 1u);
          }
          const uint32_t pos = s_fbase + recA + h;
          if (pos < q.fifo_cap) {
            Lr1Retained row;
            row.ts = r.ts; row.vidx = vidx; row.speed = (uint16_t)r.speed; row.xway = (uint16_t)r.xway;
            row.seg = (uint16_t)r.seg; row.lane = (uint8_t)r.lane; row.dir = (uint8_t)r.dir;
            __stcs(reinterpret_cast<uint4*>(q.fifo[s_fcur] + pos), *reinterpret_cast<const uint4*>(&row));
          } else if (vidx != kEmpty32) {
            atomicExch(&q.state->fifo_overflow, 1u);
            cnt.overflow++;
          }
          continue;
        }
        if (!valid) { cnt.bad++; continue; }
        if (wm_prev != 0 && (unsigned long long)r.ts + 1ull < wm_prev) { cnt.late++; continue; }   // R7
        cnt.ts_min = min(cnt.ts_min, r.ts);
        cnt.ts_max1 = max(cnt.ts_max1, r.ts + 1u);
        const uint32_t p = pane_of(r.ts, q.S, q.div_magic);
        if (!kLR1) {
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
    }
    __syncthreads();   // stage s fully consumed
    if (tid == 0 && t + kLrStages < t1) lr_issue<kLR1>(a.segs, iss, t + kLrStages, buf, &full[s]);
  }

  if (!kLR1) {
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

}  // namespace

// Load every kernel of this file now (CUDA 12 loads kernels lazily, at first launch, and a
// lazy load waits for the device: a first launch behind a running spin-wait kernel of another
// handle — the multi-GPU device barriers on a shared GPU — would wait for that spin to time
// out).  Called once per process from lms_query_create.
void preload_lr_kernels() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_lr_agg<kLR2S>);
  cudaFuncGetAttributes(&fa, k_lr_agg<kLR1S>);
}

int lr_agg_ctas(const QueryDev& q) {
  static int nsm = -1;
  if (nsm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  (void)q;
  return nsm * 2;
}

size_t lr_agg_smem(const QueryDev& q) {
  const bool lr1 = (q.kind == kLR1S || q.kind == kLR1T);
  return (size_t)kLrStages * kLrTileBytes + (lr1 ? 0 : (size_t)4 * q.K * sizeof(uint32_t));
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
    case kLR1T:
      e = set_smem_once((const void*)k_lr_agg<kLR1S>, (int)smem);
      if (e != cudaSuccess) return e;
      k_lr_agg<kLR1S><<<grid, kLrThreads, smem, st>>>(a);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace lms
