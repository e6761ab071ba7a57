// Window close / slide (all queries) and LR1 pane eviction.
//
// PAPER.md Table IV windows: "[range R slide S]", tumbling when SlideTime = 0
// (Table I).  Emission rule and window alignment: DESIGN.md readings R5, R7, R19.
// An instance k = [kS, kS+R) is the union of panes k .. k+R/S-1; a pane is evicted as soon
// as the last instance containing it has been emitted (pane state carried between batches).
//
// One launch per micro-batch.  Every CTA owns a slice of the key space and, for that slice,
//   1. (LR2 with LMS_LR2_PARTIALS=1 only, an A/B path) merges the aggregate kernel's per-CTA
//      partial tables into the pane accumulators; by default the aggregate CTAs add directly,
//   2. emits every instance k in [next_k, k_last] (k_last = floor((W-R)/S), flush:
//      floor(W/S)): SUM/COUNT over its panes, AVG = SUM/COUNT in fp64, HAVING avg < 40.0
//      (LR2), ORDER BY SUM(cpu) rank (CM1), one row per non-empty group — CM2's 16 striped
//      copies per pane are summed by 32 warps over (pane, stripe) pairs (close_striped),
//   3. zeroes its slice of every pane <= k_last.
// A batch that closes nothing goes straight to the ticket: one round trip for the window
// range, the last CTA advances the state and writes the report.
// The slices are disjoint, so no grid barrier is needed; the last CTA (atomic ticket) frees
// the evicted pane slots, rebuilds the pane table, advances next_k / the watermark snapshot
// and writes the batch report.  LR1 instead probes the retained rows of each closing
// instance's newest slide against the summed per-pane vehicle counts (bag multiplicity,
// reading R8), compacts the row FIFO, and a second small kernel frees the panes.
#include "../../include/lmstream.h"
#include "common.cuh"

namespace lms {
namespace {

constexpr int kCloseThreads = 256;
constexpr int kCloseThreadsCm2 = 1024;  // k_close_agg for CM2S: 32 warps over (pane, stripe) pairs
constexpr int kMaxPartEntries = 1024;   // 2 * aggregate CTAs
constexpr int kMaxG = 4;                // distinct pane slots merged in smem per batch
constexpr int kMaxSlice = 64;           // keys per close CTA (LR2: 200 * xways / 148 <= 22)
constexpr int kMaxH = 4096;             // pane table entries (P <= 1024)

struct CloseArgs {
  QueryDev q;
  int flush;
};

struct WinRange {
  long long nk, k_last;
  bool any;   // data was ever seen
};

__device__ __forceinline__ WinRange win_range(const QueryDev& q, int flush) {
  const DevState* st = q.state;
  WinRange w{0, -1, false};
  // the four state words in one round trip (no load behind a branch on another)
  const unsigned long long wm = st->wm;
  const uint32_t nk_valid = st->next_k_valid;
  const unsigned long long ts_min = st->ts_min;
  const long long next_k = st->next_k;
  if (wm == 0) return w;
  w.any = true;
  const long long W = (long long)wm - 1;
  if (nk_valid) w.nk = next_k;
  else w.nk = floor_div_S((long long)ts_min - (long long)q.R, q.S, q.div_magic) + 1;
  w.k_last = floor_div_S(flush ? W : W - (long long)q.R, q.S, q.div_magic);
  return w;
}

// Resolve the accumulator slots of instance k's panes into smem (kEmpty32: pane never seen),
// and at slots[ppw] the pane just past the instance (the only live pane a key can have beyond
// the last closing instance: see reclaim below).
__device__ __forceinline__ void window_slots(const QueryDev& q, long long k, uint32_t* slots) {
  __syncthreads();
  for (uint32_t j = threadIdx.x; j <= q.ppw; j += blockDim.x) slots[j] = find_slot(q, k + j);
  __syncthreads();
}

// Key-state eviction (dictionary kinds, single GPU): a key whose counts are zero in every pane
// that is still live after this close has no state left — its dictionary entry becomes a
// tombstone and its dense index goes on the free stack for the next new key, so the key
// capacity bounds the keys live in the window, not the keys ever seen (a churning jobId
// stream).  Runs in the close kernels only, never concurrently with dictionary lookups.
__device__ void reclaim_key(const QueryDev& q, uint32_t idx) {
  const unsigned long long key = q.dict.key_by_idx[idx];
  if (key == kEmpty64) return;                              // already free
  unsigned long long h = fmix64(key) & q.dict.cap_mask;
  for (unsigned long long n = 0; n <= q.dict.cap_mask; n++) {
    unsigned long long* ent = q.dict.keys + 2 * h;
    const unsigned long long k = *ent;
    if (k == key) { *ent = kTomb64; break; }
    if (k == kEmpty64) break;
    h = (h + 1) & q.dict.cap_mask;
  }
  q.dict.key_by_idx[idx] = kEmpty64;
  q.dict.free_idx[atomicAdd(&q.state->kfree_top, 1)] = idx;
  atomicAdd(&q.state->n_tomb, 1u);
}

// Whole CTA: rebuild the dictionary's hash table from the live keys (drops the tombstones;
// every live key keeps its dense index).
// Dictionary rebuild policy: above a quarter of the entries tombstoned, the batch report asks
// the host for the grid-wide rebuild (k_dict_clear + k_dict_reinsert, enqueued before the next
// batch: ~tens of microseconds for 2^21 entries); only above half does the closing CTA rebuild
// the table itself (one CTA: milliseconds — a safety net, e.g. for pipelined handles).
__device__ __forceinline__ bool dict_wants_rehash(const QueryDev& q, const DevState* st) {
  return st->n_tomb > (uint32_t)((q.dict.cap_mask + 1) / 4);
}
__device__ __forceinline__ bool dict_must_rehash(const QueryDev& q, const DevState* st) {
  return st->n_tomb > (uint32_t)((q.dict.cap_mask + 1) / 2);
}

__device__ void dict_rehash_cta(const QueryDev& q) {
  const unsigned long long cap = q.dict.cap_mask + 1;
  for (unsigned long long i = threadIdx.x; i < cap; i += blockDim.x) {
    q.dict.keys[2 * i] = kEmpty64;
    q.dict.keys[2 * i + 1] = kEmpty64;
  }
  __syncthreads();
  const uint32_t hwm = min(q.state->n_keys, q.dict.max_keys);
  for (uint32_t idx = threadIdx.x; idx < hwm; idx += blockDim.x) {
    const unsigned long long key = q.dict.key_by_idx[idx];
    if (key == kEmpty64) continue;
    unsigned long long h = fmix64(key) & q.dict.cap_mask;
    while (atomicCAS(q.dict.keys + 2 * h, kEmpty64, key) != kEmpty64) h = (h + 1) & q.dict.cap_mask;
    reinterpret_cast<unsigned int*>(q.dict.keys + 2 * h + 1)[0] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) q.state->n_tomb = 0;
}

__device__ __forceinline__ unsigned long long row_slot(DevState* st, bool want) {
  // warp-aggregated append to the result buffer
  const uint32_t act = __activemask();
  const uint32_t m = __ballot_sync(act, want);
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long base = 0;
  const int leader = m ? __ffs(m) - 1 : 0;
  if (m && (int)lane == leader) base = atomicAdd(&st->rows, (unsigned long long)__popc(m));
  base = __shfl_sync(act, base, leader);
  return base + __popc(m & ((1u << lane) - 1u));
}

// Whole-CTA: free slots holding panes <= upto and rebuild the pane hash table (P <= 1024).
__device__ void evict_rebuild_cta(const QueryDev& q, long long upto) {
  __shared__ uint32_t s_pane[1024];
  __shared__ uint32_t s_key[kMaxH];
  __shared__ int s_need;
  const uint32_t P = q.P, H = q.H_mask + 1;
  if (threadIdx.x == 0) s_need = q.state->pane_fail ? 1 : 0;
  __syncthreads();
  for (uint32_t s = threadIdx.x; s < P; s += blockDim.x) {
    uint32_t p = q.slot_pane[s];
    if (p != kEmpty32 && (long long)p <= upto) { p = kEmpty32; q.slot_pane[s] = kEmpty32; s_need = 1; }
    s_pane[s] = p;
  }
  __syncthreads();
  if (!s_need) return;
  for (uint32_t h = threadIdx.x; h < H; h += blockDim.x) { s_key[h] = kEmpty32; q.pane_slot[h] = kEmpty32; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int top = 0;
    for (uint32_t s = 0; s < P; s++) {
      const uint32_t p = s_pane[s];
      if (p == kEmpty32) { q.free_stack[top++] = s; continue; }
      uint32_t h = pane_hash(p, q.H_mask);
      while (s_key[h] != kEmpty32) h = (h + 1) & q.H_mask;
      s_key[h] = p;
      q.pane_slot[h] = s;
    }
    q.state->free_top = top;
    q.state->pane_fail = 0;
  }
  __syncthreads();
  for (uint32_t h = threadIdx.x; h < H; h += blockDim.x) q.pane_key[h] = s_key[h];
}

// Last CTA (all threads): state advance + report.
__device__ void finish(const QueryDev& q, const WinRange& w, bool swap_fifo = true) {
  DevState* st = q.state;
  const bool lr1 = (q.kind == kLR1S || q.kind == kLR1T);
  if (q.kind == kLR2S)
    for (uint32_t i = threadIdx.x; i < 2 * q.n_agg_ctas; i += blockDim.x) q.part_tag[i] = kEmpty64;
  // LR1: k_lr1_evict frees the slots.  A batch that closes nothing has nothing to evict: its
  // k_last is the previous close's, whose panes are gone, and a kept record's pane lies past it
  // (ts >= the previous watermark) — unless a pane claim failed, which the rebuild retries.
  if (w.any && !lr1 && (w.k_last >= w.nk || *(volatile uint32_t*)&st->pane_fail)) evict_rebuild_cta(q, w.k_last);
  {   // tombstones above a quarter of the table: rebuild it (LR1: in k_lr1_evict)
    __shared__ int s_rehash;
    if (threadIdx.x == 0) {
      const bool dk = q.kind == kCM2S && q.world == 1;
      s_rehash = dk && dict_must_rehash(q, st);
      q.report->rehash_req = (dk && !s_rehash && dict_wants_rehash(q, st)) ? 1u : 0u;
    }
    __syncthreads();
    if (s_rehash) dict_rehash_cta(q);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kMaxWorld; i += blockDim.x) {   // bucket counters (multi-GPU)
    st->owner_count[i] = 0;
    st->owner_cursor[i] = 0;
  }
  if (threadIdx.x == 0) {
    // every field is read up front, in one round trip: interleaved with the report stores
    // (which may alias as far as the compiler knows) each load would wait for the last one
    const unsigned long long wm = st->wm, n_records = st->n_records, bad = st->bad, late = st->late,
                             overflow = st->overflow, rows = st->rows, wclosed = st->windows_closed;
    const uint32_t n_keys = st->n_keys - (uint32_t)max(st->kfree_top, 0),   // live keys
                   row_ovf = st->row_overflow, key_ovf = st->key_overflow,
                   fifo_ovf = st->fifo_overflow, fcur = st->fifo_cur, vid_rng = st->vid_range;
    long long ck_first = 0, ck_last = -1;
    unsigned long long wc = wclosed;
    if (w.any) {
      wc += (unsigned long long)(w.k_last >= w.nk ? (w.k_last - w.nk + 1) : 0);
      ck_first = w.nk;
      ck_last = w.k_last;
      st->evict_upto = w.k_last;
      st->next_k = w.k_last + 1 > w.nk ? w.k_last + 1 : w.nk;
      st->next_k_valid = 1;
    }
    if (lr1 && swap_fifo) {
      st->fifo_count[fcur] = 0;
      st->fifo_cur = fcur ^ 1u;
    }
    const unsigned long long part_rows = rows < q.row_cap ? rows : q.row_cap;
    st->close_k_first = ck_first;
    st->close_k_last = ck_last;
    st->wm_prev = wm;
    st->part_rows = part_rows;
    BatchReport* r = q.report;
    r->n_records = n_records; r->bad = bad; r->late = late; r->overflow = overflow;
    r->rows = rows; r->windows_closed = wc;
    r->watermark = wm ? (long long)wm - 1 : -1;
    r->n_keys = n_keys; r->row_overflow = row_ovf; r->key_overflow = key_ovf;
    r->fifo_overflow = fifo_ovf;
    r->vid_range = vid_rng;
    r->close_k_first = ck_first;
    r->close_k_last = ck_last;
    r->part_rows = part_rows;
    st->n_records = st->bad = st->late = st->overflow = st->rows = st->windows_closed = 0;
    st->row_overflow = 0;
    st->fifo_overflow = 0;
    st->key_overflow = 0;
    st->vid_range = 0;
    st->ts_min = kEmpty32;
    st->close_ticket = 0;
    // (no trailing fence: the next kernel on the stream sees these writes, and the host reads
    // the mapped report after the batch's end event)
  }
}

// The last CTA to arrive returns true.  publish: this CTA wrote global data the last one will
// read (the fence orders it before the arrival); a CTA that wrote nothing skips the fence.
__device__ __forceinline__ bool ticket(DevState* st, bool publish = true) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    if (publish) __threadfence();
    last = atomicAdd(&st->close_ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// LR2: merge the per-CTA partial tables (this batch) of keys [k0, k1) into the accumulators.
__device__ void merge_partials(const QueryDev& q, uint32_t k0, uint32_t k1) {
  __shared__ uint32_t s_g[kMaxG];
  __shared__ uint8_t s_gl[kMaxPartEntries];
  __shared__ uint32_t s_lo[kMaxG][kMaxSlice], s_hi[kMaxG][kMaxSlice], s_cnt[kMaxG][kMaxSlice];
  const uint32_t ne = 2 * q.n_agg_ctas, nk = k1 - k0, K = q.K;
  if (threadIdx.x < kMaxG) s_g[threadIdx.x] = kEmpty32;
  for (uint32_t i = threadIdx.x; i < kMaxG * kMaxSlice; i += blockDim.x) {
    (&s_lo[0][0])[i] = 0; (&s_hi[0][0])[i] = 0; (&s_cnt[0][0])[i] = 0;
  }
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < ne; e += blockDim.x) {
    const unsigned long long tg = q.part_tag[e];
    uint8_t gl = 0xFF;                                         // 0xFF: unused entry
    if (tg != kEmpty64) {
      const uint32_t slot = (uint32_t)(tg >> 32);
      gl = kMaxG;                                              // kMaxG: merge with global atomics
      for (int j = 0; j < kMaxG; j++) {   // read first: nearly all entries share one pane slot
        uint32_t old = *(volatile uint32_t*)&s_g[j];
        if (old == kEmpty32) old = atomicCAS(&s_g[j], kEmpty32, slot);
        if (old == kEmpty32 || old == slot) { gl = (uint8_t)j; break; }
      }
    }
    s_gl[e] = gl;
  }
  __syncthreads();
  if (nk == 0) return;
  // thread -> (key kk, entry lane le): lane le walks entries le, le+L, ... with register
  // accumulators per merged pane slot and independent (pipelined) loads
  const uint32_t L = blockDim.x / nk;
  if (threadIdx.x < L * nk) {
    const uint32_t kk = threadIdx.x % nk, le = threadIdx.x / nk;
    unsigned long long as[kMaxG] = {0, 0, 0, 0};
    uint32_t ac[kMaxG] = {0, 0, 0, 0};
    const uint32_t* base = q.part32 + k0 + kk;
#pragma unroll 4
    for (uint32_t e = le; e < ne; e += L) {
      const uint32_t gl = s_gl[e];
      const uint32_t* part = base + (size_t)(2 * e) * K;
      const uint32_t cv = gl == 0xFF ? 0u : part[K];
      const uint32_t sv = gl == 0xFF ? 0u : part[0];
      if (gl < kMaxG) {
#pragma unroll
        for (int j = 0; j < kMaxG; j++)
          if ((uint32_t)j == gl) { as[j] += sv; ac[j] += cv; }
      } else if (gl == kMaxG && cv) {                          // more than kMaxG panes: direct
        const size_t g = (size_t)(q.part_tag[e] >> 32) * K + k0 + kk;
        atomicAdd(&q.acc_sum[g], (unsigned long long)sv);
        atomicAdd(&q.acc_cnt[g], (unsigned long long)cv);
      }
    }
#pragma unroll
    for (int j = 0; j < kMaxG; j++) {
      if (!ac[j]) continue;
      const uint32_t lo = (uint32_t)as[j], old = atomicAdd(&s_lo[j][kk], lo);
      atomicAdd(&s_hi[j][kk], (uint32_t)(as[j] >> 32) + (old + lo < old ? 1u : 0u));
      atomicAdd(&s_cnt[j][kk], ac[j]);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kMaxG * nk; i += blockDim.x) {
    const uint32_t gl = i / nk, kk = i - gl * nk;
    const uint32_t slot = s_g[gl];
    if (slot == kEmpty32 || s_cnt[gl][kk] == 0) continue;
    const size_t g = (size_t)slot * K + k0 + kk;
    q.acc_sum[g] += ((unsigned long long)s_hi[gl][kk] << 32) | s_lo[gl][kk];
    q.acc_cnt[g] += s_cnt[gl][kk];
  }
}

// Shared-memory u64 accumulation as two native u32 atomics (a 64-bit shared atomicAdd is a CAS
// loop): the carry out of the low word is added to the high word by the add that produced it.
__device__ __forceinline__ void smem_add64(uint32_t* lo, uint32_t* hi, unsigned long long v) {
  if (v == 0) return;
  const uint32_t vl = (uint32_t)v, old = atomicAdd(lo, vl);
  atomicAdd(hi, (uint32_t)(v >> 32) + (old + vl < old ? 1u : 0u));
}

// CM2 emission of instance k for keys [k0, k1): a key's accumulators are spread over
// q.stripes copies per pane (the aggregate's striped RED.64s), so one thread per key would walk
// ppw * stripes loads one round trip at a time (~400 per key at R/S = 12, 16 stripes: a closing
// batch's close took ~60 us).  The CM2 close runs 1024-thread CTAs: the CTA takes its keys 64
// at a time, lane l of warp w holds keys base + l and base + 32 + l and walks the (pane,
// stripe) pairs w, w + W, ... of the instance (coalesced over keys, 4 independent loads per
// pair, unrolled), the warps' partial sums meet in shared memory (u32-pair atomics), and
// threads 0..63 emit one key each.
__device__ __forceinline__ void close_striped(const QueryDev& q, const WinRange& w, long long k, uint32_t k0, uint32_t k1,
                                              const uint32_t* wslots, bool reclaim, lms_agg_row* rows) {
  constexpr uint32_t KB = 64;
  __shared__ uint32_t r_lo[4][KB], r_hi[4][KB];              // sum, count, first-pane count, next-pane count
  DevState* st = q.state;
  const uint32_t W = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool last = reclaim && k == w.k_last;
  const uint32_t ssh = __ffs(q.stripes) - 1, smask = q.stripes - 1;   // stripes: a power of two
  const uint32_t npairs = q.ppw << ssh;
  const uint32_t gx = wslots[q.ppw];                           // the pane after the instance
  for (uint32_t kb = k0; kb < k1; kb += KB) {
    for (uint32_t i = threadIdx.x; i < 4 * KB; i += blockDim.x) { (&r_lo[0][0])[i] = 0; (&r_hi[0][0])[i] = 0; }
    __syncthreads();
    const uint32_t key0 = kb + lane, key1 = kb + 32 + lane;
    const bool v0 = key0 < k1, v1 = key1 < k1;
    unsigned long long s0 = 0, c0 = 0, f0 = 0, x0 = 0, s1 = 0, c1 = 0, f1 = 0, x1 = 0;
#pragma unroll 4
    for (uint32_t pr = warp; pr < npairs; pr += W) {
      const uint32_t j = pr >> ssh, g = wslots[j];
      const bool u = g != kEmpty32;
      const size_t gi = ((size_t)g * q.stripes + (pr & smask)) * q.K;
      const unsigned long long a0 = (u && v0) ? q.acc_sum[gi + key0] : 0ull, n0 = (u && v0) ? q.acc_cnt[gi + key0] : 0ull;
      const unsigned long long a1 = (u && v1) ? q.acc_sum[gi + key1] : 0ull, n1 = (u && v1) ? q.acc_cnt[gi + key1] : 0ull;
      s0 += a0; c0 += n0; s1 += a1; c1 += n1;
      if (j == 0) { f0 += n0; f1 += n1; }
    }
    if (last && gx != kEmpty32)
      for (uint32_t sp = warp; sp < q.stripes; sp += W) {
        const size_t gi = ((size_t)gx * q.stripes + sp) * q.K;
        if (v0) x0 += q.acc_cnt[gi + key0];
        if (v1) x1 += q.acc_cnt[gi + key1];
      }
    smem_add64(&r_lo[0][lane], &r_hi[0][lane], s0);
    smem_add64(&r_lo[1][lane], &r_hi[1][lane], c0);
    smem_add64(&r_lo[2][lane], &r_hi[2][lane], f0);
    smem_add64(&r_lo[3][lane], &r_hi[3][lane], x0);
    smem_add64(&r_lo[0][32 + lane], &r_hi[0][32 + lane], s1);
    smem_add64(&r_lo[1][32 + lane], &r_hi[1][32 + lane], c1);
    smem_add64(&r_lo[2][32 + lane], &r_hi[2][32 + lane], f1);
    smem_add64(&r_lo[3][32 + lane], &r_hi[3][32 + lane], x1);
    __syncthreads();
    if (threadIdx.x < KB) {
      const uint32_t i = threadIdx.x, key = kb + i;
      const unsigned long long s = ((unsigned long long)r_hi[0][i] << 32) | r_lo[0][i];
      const unsigned long long c = ((unsigned long long)r_hi[1][i] << 32) | r_lo[1][i];
      const unsigned long long cf = ((unsigned long long)r_hi[2][i] << 32) | r_lo[2][i];
      const unsigned long long cx = ((unsigned long long)r_hi[3][i] << 32) | r_lo[3][i];
      // the last closing instance decides key eviction: after this close the live panes are
      // k_last + 1 .. k_last + ppw (the watermark is below (k_last + 1) S + R)
      const bool dead = last && key < k1 && (c - cf) + cx == 0;
      const bool want = key < k1 && c > 0;
      const double sum = (double)s / 1e6;                     // SUM(cpu) from the exact fixed-point sum (R20)
      const double avg = want ? sum / (double)c : 0.0;
      const unsigned long long pos = row_slot(st, want);
      if (want) {
        if (pos < q.row_cap) {
          lms_agg_row r;
          r.win_start_s = k * (long long)q.S;
          r.win_end_s = r.win_start_s + (long long)q.R;
          r.count = c; r.sum_fixed = s; r.sum = sum; r.avg = avg; r.rank = 0;
          r.key = q.dict.key_by_idx[key]; r.key_xway = r.key_dir = r.key_seg = 0;
          rows[pos] = r;
        } else {
          atomicExch(&st->row_overflow, 1u);
        }
      }
      if (dead) reclaim_key(q, key);                          // (after its row: the row reads key_by_idx)
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kCloseThreadsCm2) k_close_agg(const CloseArgs a) {
  const QueryDev& q = a.q;
  DevState* st = q.state;
  const WinRange w = win_range(q, a.flush);

  // Most batches close no window (slide S > batch span): nothing to merge (CM: the aggregate
  // pass wrote the pane accumulators directly), emit or evict.  The state is still advanced by
  // the LAST CTA to arrive (ticket), never by a fixed CTA: finish() rewrites next_k /
  // next_k_valid / ts_min, and a CTA that had not read them yet could otherwise see a torn
  // snapshot (next_k_valid = 1 with a stale next_k) and close instances that do not exist.
  if ((q.kind != kLR2S || q.lr2_direct) && !(w.any && w.k_last >= w.nk)) {
    if (ticket(st, false)) finish(q, w);
    return;
  }

  const uint32_t K = (q.kind == kCM2S) ? min(st->n_keys, q.K) : q.K;
  const uint32_t k0 = (uint32_t)((unsigned long long)K * blockIdx.x / gridDim.x);
  const uint32_t k1 = (uint32_t)((unsigned long long)K * (blockIdx.x + 1) / gridDim.x);
  const uint32_t P = q.P;
  __shared__ uint32_t wslots[257];   // R/S <= 256, + the pane after the instance
  const bool reclaim = q.kind == kCM2S && q.world == 1;

  // 1. merge LR2 partials of this batch into the pane accumulators (my key slice)
  if (q.kind == kLR2S && !q.lr2_direct) merge_partials(q, k0, k1);
  __syncthreads();

  // 2. emit closing instances
  if (w.any && w.k_last >= w.nk) {
    lms_agg_row* rows = reinterpret_cast<lms_agg_row*>(q.rows);
    for (long long k = w.nk; k <= w.k_last; k++) {
      window_slots(q, k, wslots);
      if (q.kind == kCM1S || q.kind == kCM1T) {
        // single CTA (grid = 1); K <= 10 categories; ORDER BY SUM(cpu), ties by category (R9)
        __shared__ unsigned long long s_sum[10], s_cnt[10];
        if (threadIdx.x < 10) {
          unsigned long long s = 0, c = 0;
          for (uint32_t j = 0; j < q.ppw; j++) {
            const uint32_t g = wslots[j];
            if (g != kEmpty32) { s += q.acc_sum[(size_t)g * q.K + threadIdx.x];
                                 c += q.acc_cnt[(size_t)g * q.K + threadIdx.x]; }
          }
          s_sum[threadIdx.x] = s;
          s_cnt[threadIdx.x] = c;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
          const uint32_t c = threadIdx.x;
          const bool want = c < 10 && s_cnt[c] > 0;
          uint32_t rank = 0;
          if (want && q.world == 1)                             // multi-GPU: the owner ranks
            for (uint32_t j = 0; j < 10; j++)
              if (s_cnt[j] > 0 && (s_sum[j] < s_sum[c] || (s_sum[j] == s_sum[c] && j < c))) rank++;
          const unsigned long long pos = row_slot(st, want);
          if (want) {
            if (pos < q.row_cap) {
              lms_agg_row r;
              r.win_start_s = k * (long long)q.S;
              r.win_end_s = r.win_start_s + (long long)q.R;
              r.key = c; r.count = s_cnt[c]; r.sum_fixed = s_sum[c];
              r.sum = (double)s_sum[c] / 1e6;
              r.avg = r.sum / (double)s_cnt[c];
              r.key_xway = r.key_dir = r.key_seg = 0;
              r.rank = rank;
              rows[pos] = r;
            } else {
              atomicExch(&st->row_overflow, 1u);
            }
          }
        }
        continue;
      }
      if (q.stripes > 1) {   // CM2: the 16 stripes of a key split over the CTA's warps
        close_striped(q, w, k, k0, k1, wslots, reclaim, rows);
        continue;
      }
      // LR2 (one stripe): one thread per key of my slice
      for (uint32_t kb = k0; kb < k1; kb += blockDim.x) {
        const uint32_t key = kb + threadIdx.x;
        unsigned long long s = 0, c = 0, c_first = 0;
        if (key < k1) {
          for (uint32_t j = 0; j < q.ppw; j++) {
            const uint32_t g = wslots[j];
            if (g != kEmpty32)
              for (uint32_t sp = 0; sp < q.stripes; sp++) {   // (stripes > 1: CM2)
                const size_t gi = ((size_t)g * q.stripes + sp) * q.K + key;
                s += q.acc_sum[gi];
                c += q.acc_cnt[gi];
              }
            if (j == 0) c_first = c;
          }
        }
        // the last closing instance decides key eviction: after this close the live panes are
        // k_last + 1 .. k_last + ppw (the watermark is below (k_last + 1) S + R)
        bool dead = false;
        if (reclaim && k == w.k_last && key < k1) {
          unsigned long long c_live = c - c_first;
          const uint32_t gx = wslots[q.ppw];
          if (gx != kEmpty32)
            for (uint32_t sp = 0; sp < q.stripes; sp++) c_live += q.acc_cnt[((size_t)gx * q.stripes + sp) * q.K + key];
          dead = c_live == 0;
        }
        bool want = c > 0;
        double sum, avg;
        if (q.kind == kLR2S) {
          sum = (double)s;                 // integer speed sum, exact below 2^53
          avg = want ? sum / (double)c : 0.0;
          // HAVING (avgSpeed < 40.0); multi-GPU partial rows are filtered by the owner
          want = want && (q.world > 1 || avg < 40.0);
        } else {
          sum = (double)s / 1e6;           // SUM(cpu) from the exact fixed-point sum (R20)
          avg = want ? sum / (double)c : 0.0;
        }
        const unsigned long long pos = row_slot(st, want);
        if (want) {
          if (pos < q.row_cap) {
            lms_agg_row r;
            r.win_start_s = k * (long long)q.S;
            r.win_end_s = r.win_start_s + (long long)q.R;
            r.count = c; r.sum_fixed = s; r.sum = sum; r.avg = avg; r.rank = 0;
            if (q.kind == kLR2S) {
              r.key = key; r.key_xway = key / 200u; r.key_dir = (key / 100u) % 2u; r.key_seg = key % 100u;
            } else {
              r.key = q.dict.key_by_idx[key]; r.key_xway = r.key_dir = r.key_seg = 0;
            }
            rows[pos] = r;
          } else {
            atomicExch(&st->row_overflow, 1u);
          }
        }
        if (dead) reclaim_key(q, key);          // (after its row: the row reads key_by_idx)
      }
    }
  }

  // 3. zero my key slice of every pane whose last instance has been emitted
  if (w.any) {
    const uint32_t kk0 = (q.kind == kCM1S || q.kind == kCM1T) ? 0 : k0;
    const uint32_t kk1 = (q.kind == kCM1S || q.kind == kCM1T) ? q.K : k1;
    __shared__ uint32_t s_ev[1024];                            // evicted slots (P <= 1024)
    __shared__ uint32_t s_nev;
    __syncthreads();
    if (threadIdx.x == 0) s_nev = 0;
    __syncthreads();
    for (uint32_t g = threadIdx.x; g < P; g += blockDim.x) {   // compact the evicted slots
      const uint32_t p = q.slot_pane[g];
      if (p != kEmpty32 && (long long)p <= w.k_last) s_ev[atomicAdd(&s_nev, 1u)] = g;
    }
    __syncthreads();
    const uint32_t nev = s_nev;
    // (key, stripe) pairs over the whole CTA: warp w zeroes stripes w, w + W, ... of the slice
    // (one stripe: every thread over the keys, as before)
    const uint32_t W = q.stripes > 1 ? blockDim.x / 32 : 1, wid = q.stripes > 1 ? threadIdx.x >> 5 : 0;
    const uint32_t t0 = q.stripes > 1 ? (threadIdx.x & 31) : threadIdx.x, tn = q.stripes > 1 ? 32 : blockDim.x;
    for (uint32_t i = 0; i < nev; i++) {
      const size_t g = s_ev[i];
      for (uint32_t sp = wid; sp < q.stripes; sp += W)
        for (uint32_t k = kk0 + t0; k < kk1; k += tn) {
          q.acc_sum[(g * q.stripes + sp) * q.K + k] = 0;
          q.acc_cnt[(g * q.stripes + sp) * q.K + k] = 0;
        }
    }
  }
  if (ticket(st)) finish(q, w);
}

// LR1 window counts of the first kLr1Wc instances a close emits: wc[i][v] = the count of
// vehicle index v over instance (nk + i)'s panes, one dense pass over the panes' count arrays
// (L2-resident: ppw x 4 B x vehicles), so that the probe reads one count per row instead of
// ppw gathers.  Launched before k_close_lr1 (same window range: the state is not advanced
// until k_close_lr1's last CTA); a batch that closes nothing returns at once.
constexpr uint32_t kLr1Wc = 4;           // instances with precomputed window counts
constexpr uint32_t kLr1WcMaxPpw = 64;    // R/S up to this (more: the probe sums the panes itself)
__device__ __forceinline__ uint32_t lr1_wc_instances(const QueryDev& q, const WinRange& w) {
  if (!(w.any && w.k_last >= w.nk) || q.lr1_wc == nullptr || q.world != 1 || q.ppw > kLr1WcMaxPpw) return 0;
  return (uint32_t)min(w.k_last - w.nk + 1, (long long)kLr1Wc);
}
__global__ void __launch_bounds__(kCloseThreads) k_lr1_wcache(const CloseArgs a) {
  const QueryDev& q = a.q;
  const WinRange w = win_range(q, a.flush);
  const uint32_t nI = lr1_wc_instances(q, w);
  if (nI == 0) return;
  __shared__ uint32_t sl[kLr1Wc][kLr1WcMaxPpw];
  for (uint32_t x = threadIdx.x; x < nI * q.ppw; x += blockDim.x)
    sl[x / q.ppw][x % q.ppw] = find_slot(q, w.nk + x / q.ppw + x % q.ppw);
  __syncthreads();
  const uint32_t nv = q.lr1_dense ? q.K : min(q.state->n_keys, q.K);
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t i = 0; i < nI; i++)
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nv; v += stride) {
      uint32_t m = 0;
      for (uint32_t j = 0; j < q.ppw; j++) {
        const uint32_t g = sl[i][j];
        if (g != kEmpty32) m += __ldcg(&q.acc_cnt32[(size_t)g * q.K + v]);
      }
      q.lr1_wc[(size_t)i * q.K + v] = m;
    }
}

// LR1: probe retained rows whose pane is the newest slide of a closing instance.
constexpr int kLr1Items = 2;             // retained rows per thread and iteration
constexpr int kLr1SlotCache = 1024;      // panes whose slots a CTA resolves up front
constexpr int kLr1MaxPpw = 8;
__global__ void __launch_bounds__(kCloseThreads) k_close_lr1(const CloseArgs a) {
  const QueryDev& q = a.q;
  DevState* st = q.state;
  const WinRange w = win_range(q, a.flush);
  // no instance closes (most batches): the retained rows all stay — leave the FIFO as it is
  // instead of copying every row into the other FIFO; the last CTA to arrive advances the
  // state (after every CTA has read it: see k_close_agg)
  if (!(w.any && w.k_last >= w.nk)) {
    if (ticket(st)) finish(q, w, false);
    return;
  }
  const uint32_t cur = st->fifo_cur;
  const uint32_t n = min((unsigned long long)st->fifo_count[cur], q.fifo_cap);
  const Lr1Retained* src = q.fifo[cur];
  Lr1Retained* dst = q.fifo[cur ^ 1u];
  lms_lr1_row* rows = reinterpret_cast<lms_lr1_row*>(q.rows);
  // accumulator slots of the panes the closing instances span, resolved once per CTA (a row of
  // instance k sums panes k .. k+ppw-1; outside the cached span: per-row pane-table lookups)
  __shared__ uint32_t s_slot[kLr1SlotCache + kLr1MaxPpw];
  const long long pbase = w.nk;
  const long long pspan = w.k_last + (long long)q.ppw - pbase;
  const bool cached = pspan <= kLr1SlotCache;
  if (cached)
    for (uint32_t j = threadIdx.x; j < (uint32_t)pspan; j += blockDim.x) s_slot[j] = find_slot(q, pbase + j);
  __shared__ uint32_t s_wtot[kCloseThreads / 32], s_woff[kCloseThreads / 32];
  __shared__ unsigned long long s_rbase;
  __shared__ uint32_t s_fbase;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t nwc = lr1_wc_instances(q, w);              // instances with window counts
  const uint32_t per_cta = blockDim.x * kLr1Items;
  const uint32_t iters = (n + per_cta * gridDim.x - 1) / (per_cta * gridDim.x);
  // the next iteration's retained rows are loaded one iteration ahead (their DRAM latency
  // overlaps this iteration's gathers, appends and stores); holes / past-the-end: vidx = none
  uint4 nxt[kLr1Items];
  auto load_rows = [&](uint32_t it) {
    const uint32_t base = (it * gridDim.x + blockIdx.x) * per_cta;
#pragma unroll
    for (int i = 0; i < kLr1Items; i++) {
      const uint32_t idx = base + i * blockDim.x + threadIdx.x;   // coalesced 16 B loads
      // read once: streaming load (the FIFO is not re-read from L2)
      nxt[i] = idx < n ? __ldcs(reinterpret_cast<const uint4*>(src + idx)) : make_uint4(0u, kEmpty32, 0u, 0u);
    }
  };
  if (iters) load_rows(0);
  for (uint32_t it = 0; it < iters; it++) {
    Lr1Retained r[kLr1Items];
#pragma unroll
    for (int i = 0; i < kLr1Items; i++) r[i] = *reinterpret_cast<const Lr1Retained*>(&nxt[i]);
    if (it + 1 < iters) load_rows(it + 1);
    long long kk[kLr1Items];
    uint32_t m[kLr1Items];
    uint32_t emit = 0, keep = 0;     // bit i: item i
#pragma unroll
    for (int i = 0; i < kLr1Items; i++) {
      m[i] = 0; kk[i] = 0;
      {
        if (r[i].vidx != kEmpty32) {          // (holes: records the aggregate pass dropped)
          const long long p = (long long)pane_of(r[i].ts, q.S, q.div_magic);
          kk[i] = p - (long long)q.ppw + 1;   // instance whose newest slide is pane p
          if (kk[i] <= w.k_last) emit |= 1u << i; else keep |= 1u << i;
        }
      }
    }
    // warp-aggregated appends, item-major so that every store instruction writes consecutive
    // rows: one atomic per warp and iteration on each cursor
    uint32_t em[kLr1Items], km[kLr1Items], ne = 0, nk = 0;
#pragma unroll
    for (int i = 0; i < kLr1Items; i++) {
      em[i] = __ballot_sync(0xffffffffu, emit >> i & 1u);
      km[i] = __ballot_sync(0xffffffffu, keep >> i & 1u);
      ne += __popc(em[i]); nk += __popc(km[i]);
    }
    // CTA-wide appends: warp totals -> thread 0 -> one atomic per cursor per CTA and iteration
    // (per-warp atomics on the two global cursors were the probe's main serialisation)
    const uint32_t warp = threadIdx.x >> 5;
    if (lane == 0) s_wtot[warp] = ne | (nk << 16);          // <= 32 * kLr1Items rows each per warp
    __syncthreads();
    // thread 0 reserves the CTA's rows; the reservations' latency overlaps the gathers below
    // (their results are only needed by the stores)
    unsigned long long res_rows = 0;
    uint32_t res_fifo = 0;
    if (threadIdx.x == 0) {
      uint32_t e_acc = 0, k_acc = 0;
      for (uint32_t wi = 0; wi < blockDim.x / 32u; wi++) {
        const uint32_t t = s_wtot[wi];
        s_woff[wi] = e_acc | (k_acc << 16);
        e_acc += t & 0xFFFFu;
        k_acc += t >> 16;
      }
      res_rows = e_acc ? atomicAdd(&st->rows, (unsigned long long)e_acc) : 0ull;
      res_fifo = k_acc ? atomicAdd(&st->fifo_count[cur ^ 1u], k_acc) : 0u;
    }
    // multiplicity: the vehicle's count over the instance's panes.  Common case: the window
    // counts k_lr1_wcache precomputed — one L2 load per row, all items' loads back to back.
    // Otherwise the row sums its instance's pane counts itself (cached slots or table lookups).
    uint32_t wc_mask = 0;
#pragma unroll
    for (int i = 0; i < kLr1Items; i++) {
      const long long off = kk[i] - pbase;
      if ((emit >> i & 1u) && off >= 0 && off < (long long)nwc) {
        wc_mask |= 1u << i;
        m[i] = __ldcg(&q.lr1_wc[(size_t)off * q.K + r[i].vidx]);
      }
    }
    const uint32_t slow_mask = emit & ~wc_mask;
    if (slow_mask) {
      for (int i = 0; i < kLr1Items; i++) {
        if (!(slow_mask >> i & 1u)) continue;
        const long long off = kk[i] - pbase;
        for (uint32_t j = 0; j < q.ppw; j++) {
          const uint32_t g = (cached && off >= 0) ? s_slot[off + j] : find_slot(q, kk[i] + j);
          if (g != kEmpty32) m[i] += __ldcg(&q.acc_cnt32[(size_t)g * q.K + r[i].vidx]);
        }
      }
    }
    // vehicle ids of the emitted rows (dictionary: one gather each, issued back to back)
    unsigned long long veh[kLr1Items];
#pragma unroll
    for (int i = 0; i < kLr1Items; i++)
      veh[i] = (emit >> i & 1u) ? (q.lr1_dense ? (unsigned long long)r[i].vidx : __ldcg(&q.dict.key_by_idx[r[i].vidx])) : 0ull;
    if (threadIdx.x == 0) { s_rbase = res_rows; s_fbase = res_fifo; }
    __syncthreads();
    const uint32_t wo = s_woff[warp];
    unsigned long long rbase = s_rbase + (wo & 0xFFFFu);
    uint32_t fbase = s_fbase + (wo >> 16);
#pragma unroll
    for (int i = 0; i < kLr1Items; i++) {
      if (emit >> i & 1u) {
        const unsigned long long pos = rbase + __popc(em[i] & lt);
        if (pos < q.row_cap) {
          lms_lr1_row o;
          o.win_start_s = kk[i] * (long long)q.S;
          o.vehicle = veh[i];
          o.ts = r[i].ts; o.multiplicity = m[i]; o.speed = r[i].speed; o.xway = r[i].xway;
          o.segment = r[i].seg; o.lane = r[i].lane; o.dir = r[i].dir;
          // streaming stores: 320 MB of rows per 10M probes must not evict the count tables
          const uint4* ov = reinterpret_cast<const uint4*>(&o);
          __stcs(reinterpret_cast<uint4*>(rows + pos), ov[0]);
          __stcs(reinterpret_cast<uint4*>(rows + pos) + 1, ov[1]);
        } else {
          atomicExch(&st->row_overflow, 1u);
        }
      }
      if (keep >> i & 1u) dst[fbase + __popc(km[i] & lt)] = r[i];   // rows still needed
      rbase += __popc(em[i]);
      fbase += __popc(km[i]);
    }
  }
  if (ticket(st)) finish(q, w);
}

// Grid-wide dictionary rebuild (host-enqueued between batches when a report asked for it):
// clear every entry, then reinsert every live key (key_by_idx) at its index.
__global__ void __launch_bounds__(kCloseThreads) k_dict_clear(const QueryDev q) {
  const unsigned long long n = 2 * (q.dict.cap_mask + 1);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    q.dict.keys[i] = kEmpty64;
}
__global__ void __launch_bounds__(kCloseThreads) k_dict_reinsert(const QueryDev q) {
  const uint32_t hwm = min(q.state->n_keys, q.dict.max_keys);
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < hwm; idx += gridDim.x * blockDim.x) {
    const unsigned long long key = q.dict.key_by_idx[idx];
    if (key == kEmpty64) continue;
    unsigned long long h = fmix64(key) & q.dict.cap_mask;
    while (atomicCAS(q.dict.keys + 2 * h, kEmpty64, key) != kEmpty64) h = (h + 1) & q.dict.cap_mask;
    reinterpret_cast<unsigned int*>(q.dict.keys + 2 * h + 1)[0] = idx;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) q.state->n_tomb = 0;   // (no other kernel runs on it)
}

// LR1: zero the vehicle counts of evicted panes, then (last CTA) free their slots.
__global__ void __launch_bounds__(kCloseThreads) k_lr1_evict(const QueryDev q) {
  DevState* st = q.state;
  const long long upto = st->evict_upto;
  // nothing new to evict (no instance closed since the last eviction: a kept record's pane is
  // always past the last emitted instance): every CTA sees the same values and returns
  if (upto <= st->evicted_upto && !st->pane_fail) return;
  const uint32_t nk = q.lr1_dense ? q.K : min(st->n_keys, q.K);
  __shared__ uint32_t s_live[1024];           // slots of the panes that stay live (P <= 1024)
  __shared__ uint32_t s_nlive;
  if (threadIdx.x == 0) s_nlive = 0;
  __syncthreads();
  for (uint32_t g = threadIdx.x; g < q.P; g += blockDim.x) {
    const uint32_t p = q.slot_pane[g];
    if (p != kEmpty32 && (long long)p > upto) s_live[atomicAdd(&s_nlive, 1u)] = g;
  }
  __syncthreads();
  const bool reclaim = !q.lr1_dense && q.world == 1;
  for (uint32_t g = 0; g < q.P; g++) {
    const uint32_t p = q.slot_pane[g];
    if (p == kEmpty32 || (long long)p > upto) continue;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nk; k += gridDim.x * blockDim.x)
      q.acc_cnt32[(size_t)g * q.K + k] = 0;
  }
  if (reclaim) {   // key-state eviction: vehicles with no count in any live pane (see reclaim_key)
    const uint32_t nl = s_nlive;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < nk; k += gridDim.x * blockDim.x) {
      uint32_t c = 0;
      for (uint32_t i = 0; i < nl && c == 0; i++) c += q.acc_cnt32[(size_t)s_live[i] * q.K + k];
      if (c == 0) reclaim_key(q, k);
    }
  }
  if (ticket(st)) {
    evict_rebuild_cta(q, upto);
    __shared__ int s_rehash;
    if (threadIdx.x == 0) {
      s_rehash = reclaim && dict_must_rehash(q, st);
      // (the close kernel's finish wrote this batch's report before this kernel ran)
      q.report->rehash_req = (reclaim && !s_rehash && dict_wants_rehash(q, st)) ? 1u : 0u;
    }
    __syncthreads();
    if (s_rehash) dict_rehash_cta(q);
    if (threadIdx.x == 0) { st->evicted_upto = upto; st->close_ticket = 0; __threadfence(); }
  }
}

// Multi-GPU LR1 (reading R8 on row-partitioned batches): every rank probes its own newest-pane
// rows, but the multiplicity m counts the vehicle over ALL ranks' records of the window.
// k_lr1_wsum writes this rank's counts of instance k's panes into lr1_w (vehicle-indexed,
// lr1_dense), the caller all-reduces lr1_w (SUM), and k_lr1_probe emits the rows of instance k
// with m = lr1_w[vehicle].  The union over ranks equals the single-GPU rows.
__global__ void __launch_bounds__(kCloseThreads) k_lr1_wsum(const QueryDev q, long long k) {
  __shared__ uint32_t wslots[256];   // R/S <= 256
  window_slots(q, k, wslots);
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < q.K; v += gridDim.x * blockDim.x) {
    uint32_t m = 0;
    for (uint32_t j = 0; j < q.ppw; j++) {
      const uint32_t g = wslots[j];
      if (g != kEmpty32) m += q.acc_cnt32[(size_t)g * q.K + v];
    }
    q.lr1_w[v] = m;
  }
}

__global__ void __launch_bounds__(kCloseThreads) k_lr1_probe(const QueryDev q, long long k) {
  DevState* st = q.state;
  const uint32_t cur = st->fifo_cur;
  const uint32_t n = min((unsigned long long)st->fifo_count[cur], q.fifo_cap);
  const Lr1Retained* src = q.fifo[cur];
  Lr1Retained* dst = q.fifo[cur ^ 1u];
  lms_lr1_row* rows = reinterpret_cast<lms_lr1_row*>(q.rows);
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t iters = (n + stride - 1) / stride;
  for (uint32_t it = 0; it < iters; it++) {
    const uint32_t i = it * stride + blockIdx.x * blockDim.x + threadIdx.x;
    bool emit = false, keep = false;
    Lr1Retained r{};
    if (i < n && src[i].vidx != kEmpty32) {
      r = src[i];
      const long long p = (long long)pane_of(r.ts, q.S, q.div_magic);
      emit = p - (long long)q.ppw + 1 == k;      // instance whose newest slide is pane p
      keep = !emit;
    }
    const unsigned long long pos = row_slot(st, emit);
    if (emit) {
      if (pos < q.row_cap) {
        lms_lr1_row o;
        o.win_start_s = k * (long long)q.S;
        o.vehicle = r.vidx;
        o.ts = r.ts; o.multiplicity = q.lr1_w[r.vidx]; o.speed = r.speed; o.xway = r.xway;
        o.segment = r.seg; o.lane = r.lane; o.dir = r.dir;
        const uint4* ov = reinterpret_cast<const uint4*>(&o);   // two 16 B streaming stores
        __stcs(reinterpret_cast<uint4*>(rows + pos), ov[0]);
        __stcs(reinterpret_cast<uint4*>(rows + pos) + 1, ov[1]);
      } else {
        atomicExch(&st->row_overflow, 1u);
      }
    }
    const uint32_t km = __ballot_sync(0xffffffffu, keep);
    uint32_t base = 0;
    if ((threadIdx.x & 31) == 0 && km) base = atomicAdd(&st->fifo_count[cur ^ 1u], __popc(km));
    base = __shfl_sync(0xffffffffu, base, 0);
    if (keep) dst[base + __popc(km & ((1u << (threadIdx.x & 31)) - 1u))] = r;
  }
  if (ticket(st) && threadIdx.x == 0) {          // the kept rows become the live FIFO
    st->fifo_count[cur] = 0;
    st->fifo_cur = cur ^ 1u;
    st->close_ticket = 0;
    __threadfence();
  }
}

// dst[i] = sum over g of src[g][i] (the devices' LR1 window counts, read through peer memory:
// the single-handle multi-device driver's all-reduce).
struct SumSrcs {
  const uint32_t* p[kMaxWorld];
};
__global__ void __launch_bounds__(kCloseThreads) k_sum_u32(uint32_t* dst, const SumSrcs src, uint32_t G, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    uint32_t s = 0;
    for (uint32_t g = 0; g < G; g++) s += __ldcg(src.p[g] + i);
    dst[i] = s;
  }
}

}  // namespace

cudaError_t launch_sum_u32(uint32_t* dst, const uint32_t* const* srcs, uint32_t G, uint32_t n, cudaStream_t st) {
  SumSrcs a{};
  for (uint32_t g = 0; g < G && g < (uint32_t)kMaxWorld; g++) a.p[g] = srcs[g];
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  k_sum_u32<<<2 * nsm, kCloseThreads, 0, st>>>(dst, a, G, n);
  return cudaGetLastError();
}

// Load every kernel of this file now (CUDA 12 loads kernels lazily, at first launch, and a
// lazy load waits for the device: a first launch behind a running spin-wait kernel of another
// handle — the multi-GPU device barriers on a shared GPU — would wait for that spin to time
// out).  Called once per process from lms_query_create.
void preload_close_kernels() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_close_agg);
  cudaFuncGetAttributes(&fa, k_close_lr1);
  cudaFuncGetAttributes(&fa, k_lr1_wcache);
  cudaFuncGetAttributes(&fa, k_dict_clear);
  cudaFuncGetAttributes(&fa, k_dict_reinsert);
  cudaFuncGetAttributes(&fa, k_lr1_evict);
  cudaFuncGetAttributes(&fa, k_lr1_wsum);
  cudaFuncGetAttributes(&fa, k_lr1_probe);
  cudaFuncGetAttributes(&fa, k_sum_u32);
}

static int sm_count_close() {
  static int nsm = -1;
  if (nsm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return nsm;
}

int close_ctas(const QueryDev& q) {
  if (q.kind == kCM1S || q.kind == kCM1T) return 1;
  static int nsm = -1;
  if (nsm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  // LR2: ~3 keys per CTA, so each (key, entry-lane) thread walks only ~7 of the 2C partial
  // entries (the merge is load-latency bound, not bandwidth bound)
  // LR1: the closing probe is load-latency bound (two 256-thread CTAs per SM at its register count)
  // (LR2 with direct accumulator adds — the default — has no partials to merge: one CTA per SM,
  // a quarter of the ticket arrivals of a batch that closes nothing)
  return q.kind == kLR2S ? (q.lr2_direct ? nsm : 4 * nsm) : (q.kind == kLR1S || q.kind == kLR1T) ? 4 * nsm : nsm;
}

cudaError_t launch_dict_rehash(const QueryDev& q, cudaStream_t st) {
  k_dict_clear<<<4 * sm_count_close(), kCloseThreads, 0, st>>>(q);
  k_dict_reinsert<<<4 * sm_count_close(), kCloseThreads, 0, st>>>(q);
  return cudaGetLastError();
}

int close_launches(const QueryDev& q) {
  return ((q.kind == kLR1S || q.kind == kLR1T) && q.lr1_wc != nullptr && q.world == 1) ? 2 : 1;
}

cudaError_t launch_close(const QueryDev& q, int flush, cudaStream_t st) {
  CloseArgs a{q, flush};
  if (q.kind == kLR1S || q.kind == kLR1T) {
    if (q.lr1_wc != nullptr && q.world == 1) k_lr1_wcache<<<close_ctas(q), kCloseThreads, 0, st>>>(a);
    k_close_lr1<<<close_ctas(q), kCloseThreads, 0, st>>>(a);
  }
  else k_close_agg<<<close_ctas(q), q.kind == kCM2S ? kCloseThreadsCm2 : kCloseThreads, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_lr1_wsum(const QueryDev& q, long long k, cudaStream_t st) {
  k_lr1_wsum<<<close_ctas(q), kCloseThreads, 0, st>>>(q, k);
  return cudaGetLastError();
}

cudaError_t launch_lr1_probe(const QueryDev& q, long long k, cudaStream_t st) {
  k_lr1_probe<<<close_ctas(q), kCloseThreads, 0, st>>>(q, k);
  return cudaGetLastError();
}

cudaError_t launch_lr1_evict(const QueryDev& q, cudaStream_t st) {
  k_lr1_evict<<<close_ctas(q), kCloseThreads, 0, st>>>(q);
  return cudaGetLastError();
}

}  // namespace lms
