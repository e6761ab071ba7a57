// Device helpers shared by the LMStream kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "device.h"

namespace lms {

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
// mbarrier parity wait on a shared-window address (every calling lane waits)
__device__ __forceinline__ void mbar_wait_shared(uint32_t bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAITS:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAITS;\n}" ::"r"(bar), "r"(phase) : "memory");
}

// ---- mbarrier + 1-D bulk copy (TMA engine, UBLKCP) -------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n LAB_WAIT:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra LAB_WAIT;\n}" ::"r"(smem_addr(b)),
      "r"(phase)
      : "memory");
}
// global -> shared, bytes % 16 == 0, both addresses 16-byte aligned; completes on mbarrier b.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  // (no L2 evict-first hint here, unlike the CM copies: measured 3 % slower on LR2, where no
  // table competes with the stream for L2)
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(b))
      : "memory");
}

// The same with an L2 evict-first policy (read-once input competing with L2-resident tables).
__device__ __forceinline__ void bulk_g2s_evict_first(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile(
      "{\n .reg .b64 pol;\n createpolicy.fractional.L2::evict_first.b64 pol, 1.0;\n"
      " cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], pol;\n}"
      ::"r"(smem_addr(dst)), "l"(src), "r"(bytes), "r"(smem_addr(b))
      : "memory");
}

// Segment of a monotonically advancing tile index (a CTA / warp walks its tiles in order):
// tiles [base, end) belong to segment si.  O(1) per tile instead of a search.
struct SegCursor {
  int si;
  unsigned long long base, end;
  __device__ __forceinline__ void init(const SegTable& s) { si = 0; base = 0; end = s.tile_prefix[1]; }
  __device__ __forceinline__ void seek(const SegTable& s, unsigned long long tile) {
    while (tile >= end && si + 1 < s.n) { si++; base = end; end = s.tile_prefix[si + 1]; }
  }
};

// ---- arithmetic ----------------------------------------------------------------------
// pane = ts / S exactly for ts < 2^32, S <= 2^31 (magic = ceil(2^64 / S), S > 1).
__device__ __forceinline__ uint32_t pane_of(uint32_t ts, uint32_t S, unsigned long long magic) {
  return S == 1 ? ts : (uint32_t)__umul64hi((unsigned long long)ts, magic);
}

__device__ __forceinline__ long long floor_div(long long a, long long b) {
  long long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) q--;
  return q;
}

// floor(a / S) through the pane magic (pane_of: exact for 0 <= a < 2^32, and for negative a by
// floor(a / S) = -1 - floor((-a - 1) / S)); anything else: the 64-bit division.  Window ranges
// are floor_div_S of watermark / ts differences: no 64-bit division on the close's latency path.
__device__ __forceinline__ long long floor_div_S(long long a, uint32_t S, unsigned long long magic) {
  if (a >= 0 && a < (1ll << 32)) return (long long)pane_of((uint32_t)a, S, magic);
  if (a < 0 && a > -(1ll << 32)) return -(long long)pane_of((uint32_t)(-a - 1), S, magic) - 1;
  return floor_div(a, (long long)S);
}

__device__ __forceinline__ unsigned long long fmix64(unsigned long long k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

// Dense index for a newly inserted key: a recycled one (reclaimed when its key's last pane was
// evicted, reading R7 eviction) if any, else the next fresh one.  Pops run only while no
// reclaim runs (reclaims happen in the close kernels, pops in the aggregate / merge kernels).
__device__ __forceinline__ uint32_t alloc_key_index(const Dict& d, DevState* st) {
  if (*(volatile int*)&st->kfree_top > 0) {
    const int t = atomicSub(&st->kfree_top, 1) - 1;
    if (t >= 0) return d.free_idx[t];
    atomicAdd(&st->kfree_top, 1);          // lost the race for the last one
  }
  return atomicAdd_system(&st->n_keys, 1u);
}

// Dictionary lookup-or-insert: key -> dense index < max_keys; kEmpty32 on overflow.  Entries of
// reclaimed keys are tombstones (kTomb64): probes pass over them, inserts only take empty
// entries (so that two threads inserting the same key cannot end in two entries).
__device__ __forceinline__ uint32_t dict_get(const Dict& d, unsigned long long key, DevState* st) {
  unsigned long long h = fmix64(key) & d.cap_mask;
  for (unsigned long long probes = 0; probes <= d.cap_mask; probes++) {   // bounded: a full
                                                                          // table (key overflow) ends
    unsigned long long* ent = d.keys + 2 * h;
    unsigned long long k, kv;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(k), "=l"(kv) : "l"(ent));
    if (k == kEmpty64) {
      // inserts are rare (one per distinct key) and may race with peer GPUs' inserts into the
      // same dictionary (multi-GPU fused exchange, dict_get_sys): system-scope RMWs
      k = atomicCAS_system(ent, kEmpty64, key);
      if (k == kEmpty64) {     // we own the entry: allocate the index and publish it
        uint32_t idx = alloc_key_index(d, st);
        if (idx >= d.max_keys) {
          atomicExch(&st->key_overflow, 1u);
          idx = kEmpty32 - 1;   // poison: entry exists but is unusable
        } else {
          d.key_by_idx[idx] = key;
        }
        __threadfence_system();
        atomicExch_system(reinterpret_cast<unsigned int*>(ent + 1), idx);
        return idx >= d.max_keys ? kEmpty32 : idx;
      }
      kv = kEmpty32;            // someone else inserted: re-read its index below if it is ours
    }
    if (k == key) {
      uint32_t v = (uint32_t)kv;
      while (v == kEmpty32) v = *(volatile uint32_t*)(ent + 1);
      return v >= d.max_keys ? kEmpty32 : v;
    }
    h = (h + 1) & d.cap_mask;
  }
  atomicExch(&st->key_overflow, 1u);   // every entry taken by other keys: this key is dropped
  return kEmpty32;
}

// Lookup-or-insert of two keys whose first probes are issued together: the common case (both
// keys found in their home entries) costs one L2 round trip for the pair instead of two
// dependent ones; anything else (a miss, a collision, an index being published) falls back to
// dict_get.  u0 / u1: whether the key is looked up at all (kEmpty32 otherwise).
__device__ __forceinline__ void dict_get2(const Dict& d, unsigned long long k0, bool u0, unsigned long long k1,
                                          bool u1, DevState* st, uint32_t& i0, uint32_t& i1) {
  const unsigned long long* e0 = d.keys + 2 * (fmix64(k0) & d.cap_mask);
  const unsigned long long* e1 = d.keys + 2 * (fmix64(k1) & d.cap_mask);
  unsigned long long a0 = kEmpty64, b0 = kEmpty64, a1 = kEmpty64, b1 = kEmpty64;
  if (u0) asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a0), "=l"(b0) : "l"(e0));
  if (u1) asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a1), "=l"(b1) : "l"(e1));
  const bool h0 = a0 == k0 && (uint32_t)b0 != kEmpty32, h1 = a1 == k1 && (uint32_t)b1 != kEmpty32;
  i0 = !u0 ? kEmpty32 : h0 ? ((uint32_t)b0 >= d.max_keys ? kEmpty32 : (uint32_t)b0) : dict_get(d, k0, st);
  i1 = !u1 ? kEmpty32 : h1 ? ((uint32_t)b1 >= d.max_keys ? kEmpty32 : (uint32_t)b1) : dict_get(d, k1, st);
}

// ---- pane table: pane index -> accumulator slot ------------------------------------------
__device__ __forceinline__ uint32_t pane_hash(uint32_t p, uint32_t mask) { return (p * 0x9E3779B1u) & mask; }

// Accumulator slot of pane p, allocating one on first sight; kFail32 if all P slots are live.
// Called rarely (threads cache the last pane they resolved).
__device__ __forceinline__ uint32_t claim_slot(const QueryDev& q, uint32_t p) {
  uint32_t h = pane_hash(p, q.H_mask);
  for (uint32_t probes = 0; probes <= q.H_mask; probes++) {   // bounded: a full pane table ends
    uint32_t k = *(volatile uint32_t*)&q.pane_key[h];
    if (k == kEmpty32) {
      k = atomicCAS(&q.pane_key[h], kEmpty32, p);
      if (k == kEmpty32) {   // we inserted p: allocate a slot and publish it
        const int top = atomicSub(&q.state->free_top, 1) - 1;
        uint32_t s = kFail32;
        if (top >= 0) {
          s = q.free_stack[top];
          q.slot_pane[s] = p;
        } else {
          atomicAdd(&q.state->free_top, 1);
          q.state->pane_fail = 1;
        }
        __threadfence();
        atomicExch(&q.pane_slot[h], s);
        return s;
      }
    }
    if (k == p) {
      uint32_t s;
      while ((s = *(volatile uint32_t*)&q.pane_slot[h]) == kEmpty32) { }
      return s;
    }
    h = (h + 1) & q.H_mask;
  }
  q.state->pane_fail = 1;               // table full of other panes: this pane's records overflow
  return kFail32;
}

// Lookup only (no concurrent inserts may run): slot of pane p or kEmpty32.
__device__ __forceinline__ uint32_t find_slot(const QueryDev& q, long long p) {
  if (p < 0 || p > 0xFFFFFFF0ll) return kEmpty32;
  uint32_t h = pane_hash((uint32_t)p, q.H_mask);
  for (uint32_t probes = 0; probes <= q.H_mask; probes++) {
    const uint32_t k = q.pane_key[h];
    if (k == kEmpty32) return kEmpty32;
    if (k == (uint32_t)p) {
      const uint32_t s = q.pane_slot[h];
      return s == kFail32 ? kEmpty32 : s;
    }
    h = (h + 1) & q.H_mask;
  }
  return kEmpty32;
}

// Per-CTA pane slots (2, tags in smem: acc slot << 32 | pane).  Sets lslot = 0/1 (local table)
// or 2 (not local: use the global accumulators directly) and gslot = accumulator slot / kFail32.
__device__ __forceinline__ void local_slot(unsigned long long* slot_tag, const QueryDev& q, uint32_t p,
                                           uint32_t& lslot, uint32_t& gslot) {
  for (int sl = 0; sl < 2; sl++) {
    unsigned long long tg = *(volatile unsigned long long*)&slot_tag[sl];
    if (tg == kEmpty64) {
      const unsigned long long want = ((unsigned long long)claim_slot(q, p) << 32) | p;
      tg = atomicCAS(&slot_tag[sl], kEmpty64, want);
      if (tg == kEmpty64) tg = want;
    }
    if ((uint32_t)tg == p) { lslot = sl; gslot = (uint32_t)(tg >> 32); return; }
  }
  lslot = 2;
  gslot = claim_slot(q, p);
}

// ---- block reductions (blockDim multiple of 32, <= 1024) ----------------------------
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) { return __reduce_max_sync(0xffffffffu, v); }

// Per-CTA counters flushed once per CTA (one atomic per counter per CTA).
struct CtaCounters {
  unsigned long long n, bad, late, overflow;
  uint32_t ts_min, ts_max1;   // ts_max1 = max ts + 1 (0 = none)
};

// scratch: >= 1280 B of 8 B aligned shared memory the CTA no longer uses (the caller's buffers,
// so that this does not add to a kernel's static shared memory); the CTA synchronises first.
__device__ __forceinline__ void flush_counters(CtaCounters c, DevState* st, void* scratch) {
  unsigned long long* s_n = static_cast<unsigned long long*>(scratch);
  unsigned long long *s_bad = s_n + 32, *s_late = s_n + 64, *s_ovf = s_n + 96;
  uint32_t* s_min = reinterpret_cast<uint32_t*>(s_n + 128);
  uint32_t* s_max = s_min + 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  c.n = warp_sum(c.n); c.bad = warp_sum(c.bad); c.late = warp_sum(c.late); c.overflow = warp_sum(c.overflow);
  c.ts_min = warp_min_u32(c.ts_min); c.ts_max1 = warp_max_u32(c.ts_max1);
  __syncthreads();
  if (lane == 0) { s_n[w] = c.n; s_bad[w] = c.bad; s_late[w] = c.late; s_ovf[w] = c.overflow;
                   s_min[w] = c.ts_min; s_max[w] = c.ts_max1; }
  __syncthreads();
  if (w == 0) {
    unsigned long long n = lane < nw ? s_n[lane] : 0, bad = lane < nw ? s_bad[lane] : 0;
    unsigned long long late = lane < nw ? s_late[lane] : 0, ovf = lane < nw ? s_ovf[lane] : 0;
    uint32_t mn = lane < nw ? s_min[lane] : kEmpty32, mx = lane < nw ? s_max[lane] : 0;
    n = warp_sum(n); bad = warp_sum(bad); late = warp_sum(late); ovf = warp_sum(ovf);
    mn = warp_min_u32(mn); mx = warp_max_u32(mx);
    if (lane == 0) {
      if (n) atomicAdd(&st->n_records, n);
      if (bad) atomicAdd(&st->bad, bad);
      if (late) atomicAdd(&st->late, late);
      if (ovf) atomicAdd(&st->overflow, ovf);
      if (mn != kEmpty32) atomicMin(&st->ts_min, (unsigned long long)mn);
      if (mx) atomicMax(&st->wm, (unsigned long long)mx);
    }
  }
}

__device__ __forceinline__ void flush_counters(CtaCounters c, DevState* st) {
  __shared__ __align__(8) unsigned long long scratch[160];
  flush_counters(c, st, scratch);
}

}  // namespace lms
