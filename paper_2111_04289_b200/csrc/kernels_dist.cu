// Multi-GPU row partitioning: owner bucketing of partial window rows and the owner-side merge.
//
// PAPER.md: the paper's micro-batch is split into partitions processed in parallel by the
// executors and aggregated after a shuffle ("Shuffling", Table III P:751;
// "shuffle aggregate" P:962).  Here every rank (GPU) aggregates its own rows of each micro-
// batch; when instances close, each rank emits PARTIAL rows (count, exact integer sum per
// (instance, key)), the rows are exchanged by owner rank (NCCL all-to-all, dist.py) and the
// owner merges them and applies what needs the whole group: AVG, HAVING (LR2), ORDER BY rank
// (CM1).  Owner = fmix64(key) % world for LR2/CM2 (no cross-key operation); for CM1 the
// owner of an instance is k % world so that one rank sees every category of it (ORDER BY).
#include "../../include/lmstream.h"
#include "common.cuh"

namespace lms {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ uint32_t owner_of(const QueryDev& q, const lms_agg_row& r) {
  if (q.kind == kCM1S || q.kind == kCM1T) {
    const long long k = floor_div(r.win_start_s, (long long)q.S);
    const long long m = k % (long long)q.world;
    return (uint32_t)(m < 0 ? m + q.world : m);
  }
  return (uint32_t)(fmix64(r.key) % q.world);
}

__global__ void __launch_bounds__(kThreads) k_bucket_count(const QueryDev q) {
  __shared__ uint32_t s_cnt[kMaxWorld];
  DevState* st = q.state;
  const unsigned long long n = st->part_rows;
  for (uint32_t i = threadIdx.x; i < q.world; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const lms_agg_row* rows = reinterpret_cast<const lms_agg_row*>(q.rows);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x)
    atomicAdd(&s_cnt[owner_of(q, rows[i])], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < q.world; i += blockDim.x)
    if (s_cnt[i]) atomicAdd(&st->owner_count[i], s_cnt[i]);
}

__global__ void __launch_bounds__(kThreads) k_bucket_scatter(const QueryDev q) {
  __shared__ uint32_t s_off[kMaxWorld];
  DevState* st = q.state;
  const unsigned long long n = st->part_rows;
  if (threadIdx.x == 0) {
    uint32_t o = 0;
    for (uint32_t i = 0; i < q.world; i++) { s_off[i] = o; o += st->owner_count[i]; }
  }
  __syncthreads();
  if (blockIdx.x == 0)
    for (uint32_t i = threadIdx.x; i < q.world; i += blockDim.x) q.report->owner_count[i] = st->owner_count[i];
  const lms_agg_row* rows = reinterpret_cast<const lms_agg_row*>(q.rows);
  lms_agg_row* out = reinterpret_cast<lms_agg_row*>(q.send_rows);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const lms_agg_row r = rows[i];
    const uint32_t o = owner_of(q, r);
    out[s_off[o] + atomicAdd(&st->owner_cursor[o], 1u)] = r;
  }
}

// Received partial rows of instances [k_lo, k_lo + nwin) -> merge accumulators.
__global__ void __launch_bounds__(kThreads) k_merge(const QueryDev q, const lms_agg_row* rows,
                                                    unsigned long long n, long long k_lo, uint32_t nwin) {
  DevState* st = q.state;
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const lms_agg_row r = rows[i];
    const long long w = floor_div(r.win_start_s, (long long)q.S) - k_lo;
    if (w < 0 || w >= (long long)nwin) continue;
    uint32_t idx;
    if (q.kind == kCM2S) idx = dict_get(q.dict, r.key, st);
    else idx = (uint32_t)r.key;
    if (idx == kEmpty32 || idx >= q.K) { atomicAdd(&st->overflow, r.count); continue; }
    const size_t g = (size_t)w * q.K + idx;
    atomicAdd(&q.macc_sum[g], r.sum_fixed);
    atomicAdd(&q.macc_cnt[g], r.count);
  }
}

// Fused exchange: instead of all-to-all of partial rows + owner merge, every
// rank adds its partial (exact sum, count) of each (instance, key) straight into the OWNER's
// merge accumulators through peer-mapped memory (remote RED.64 over NVLink); CM2 keys are
// resolved in the owner's dictionary with remote CAS.  The caller then barriers the ranks
// and each owner finalizes (k_finalize / k_finalize_cm1, unchanged).
__device__ __forceinline__ uint32_t dict_get_sys(const Dict& d, unsigned long long key, DevState* st) {
  unsigned long long h = fmix64(key) & d.cap_mask;
  for (unsigned long long probes = 0; probes <= d.cap_mask; probes++) {   // bounded: a full
                                                                          // table (key overflow) ends
    unsigned long long* ent = d.keys + 2 * h;
    unsigned long long k, kv;
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(k), "=l"(kv) : "l"(ent));
    if (k == kEmpty64) {
      k = atomicCAS_system(ent, kEmpty64, key);
      if (k == kEmpty64) {     // we own the entry: allocate the index and publish it
        uint32_t idx = atomicAdd_system(&st->n_keys, 1u);
        if (idx >= d.max_keys) {
          atomicExch_system(&st->key_overflow, 1u);
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
  atomicExch_system(&st->key_overflow, 1u);   // every entry taken by other keys: this key is dropped
  return kEmpty32;
}

// NVLS multimem operations on a multicast address (PTX ISA multimem.*: the reduction / store is
// applied by the NVLink switch to the replica of every device in the multicast group).
__device__ __forceinline__ void mc_red_add(unsigned long long* mc, unsigned long long v) {
  asm volatile("multimem.red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
}
__device__ __forceinline__ void mc_store(unsigned long long* mc, unsigned long long v) {
  asm volatile("multimem.st.relaxed.sys.global.u64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_alias() { asm volatile("fence.proxy.alias;" ::: "memory"); }
__device__ __forceinline__ bool dense_kind(const QueryDev& q) {
  return q.kind == kLR2S || q.kind == kCM1S || q.kind == kCM1T;
}

// One partial row into the merge accumulators: NVLS (dense tables, every replica) or the owner's
// accumulators through peer memory (remote RED.64; CM2 jobIds resolved in the owner's dictionary).
__device__ __forceinline__ void push_row(const QueryDev& q, DevState* st, const lms_agg_row& r, long long w) {
  if (q.mc_sum != nullptr && dense_kind(q)) {
    const uint32_t idx = (uint32_t)r.key;
    if (idx >= q.K) { atomicAdd(&st->overflow, r.count); return; }
    const size_t g = (size_t)w * q.K + idx;
    mc_red_add(q.mc_sum + g, r.sum_fixed);
    mc_red_add(q.mc_cnt + g, r.count);
    return;
  }
  const PeerView P = q.peers[owner_of(q, r)];
  uint32_t idx;
  if (q.kind == kCM2S) idx = dict_get_sys(P.dict, r.key, P.state);
  else idx = (uint32_t)r.key;
  if (idx == kEmpty32 || idx >= q.K) { atomicAdd(&st->overflow, r.count); return; }
  const size_t g = (size_t)w * q.K + idx;
  atomicAdd_system(&P.macc_sum[g], r.sum_fixed);   // remote (peer GPU) RMW: system scope
  atomicAdd_system(&P.macc_cnt[g], r.count);
}

__global__ void __launch_bounds__(kThreads) k_p2p_push(const QueryDev q, long long k_lo, uint32_t nwin) {
  DevState* st = q.state;
  const unsigned long long n = st->part_rows;
  const lms_agg_row* rows = reinterpret_cast<const lms_agg_row*>(q.send_rows);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const lms_agg_row r = rows[i];
    const long long w = floor_div(r.win_start_s, (long long)q.S) - k_lo;
    if (w < 0 || w >= (long long)nwin) continue;
    push_row(q, st, r, w);
  }
  fence_alias();
  __threadfence_system();
}

// The instances of the last close, clamped to one merge window (async exchange: nwin == 0
// on the host side; flushes with more instances use the host-driven passes).
__device__ __forceinline__ void close_window(const QueryDev& q, long long& k_lo, uint32_t& nwin) {
  const long long k0 = q.state->close_k_first, k1 = q.state->close_k_last;
  k_lo = k0;
  nwin = k1 >= k0 ? (uint32_t)min(k1 - k0 + 1, (long long)q.Wmerge) : 0u;
}

// ---- device-side barrier of the fused exchange (no host round trip) ----------------------
// Thread 0 spins until *c >= target (bounded: ~20 s of SM clock, then the error flag is raised
// and the exchange proceeds — that batch is reported as failed, nothing hangs).  clock64 is
// the SM's own cycle counter: monotonic for the spinning thread (%globaltimer proved unusable
// for this: its first reads can jump).
__device__ __forceinline__ void spin_until(DevState* st, const unsigned int* c, unsigned int target) {
  const long long t0 = clock64();
  while (*(volatile const unsigned int*)c < target) {
    if (clock64() - t0 > 40000000000ll) { atomicExch(&st->p2p_err, 1u); break; }
    __nanosleep(256);
  }
  __threadfence_system();
}
// +1 on counter `which` (0 arrive, 1 done) of every rank, after this rank's writes are visible.
__device__ __forceinline__ void signal_all(const QueryDev& q, int which) {
  __threadfence_system();
  for (uint32_t r = 0; r < q.world; r++) {
    DevState* ps = q.peers[r].state;
    atomicAdd_system(which == 0 ? &ps->p2p_arrive : &ps->p2p_done, 1u);
  }
}

// Async fused exchange, step 1 (every CTA): wait until every owner finished the previous
// exchange's finalize (it zeroes what it reads), push this rank's partials of the last close's
// instances into the owners' accumulators; the last CTA signals arrival to every rank.
__global__ void __launch_bounds__(kThreads) k_p2p_push_async(const QueryDev q) {
  DevState* st = q.state;
  long long k_lo;
  uint32_t nwin;
  close_window(q, k_lo, nwin);
  if (nwin == 0) return;                      // no instance closed (same on every rank)
  const unsigned int gen = st->p2p_gen;       // exchanges with instances before this one
  __shared__ bool last;
  if (threadIdx.x == 0) spin_until(st, &st->p2p_done, gen * q.world);
  __syncthreads();
  const unsigned long long n = st->part_rows;
  const lms_agg_row* rows = reinterpret_cast<const lms_agg_row*>(q.send_rows);
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const lms_agg_row r = rows[i];
    const long long w = floor_div(r.win_start_s, (long long)q.S) - k_lo;
    if (w < 0 || w >= (long long)nwin) continue;
    push_row(q, st, r, w);
  }
  fence_alias();
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&st->p2p_ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (last && threadIdx.x == 0) {
    st->p2p_ticket = 0;
    signal_all(q, 0);
  }
}

// Step 2 (1 thread, before the owner's finalize): every rank has pushed.
__global__ void k_p2p_wait_arrive(const QueryDev q) {
  DevState* st = q.state;
  long long k_lo;
  uint32_t nwin;
  close_window(q, k_lo, nwin);
  if (nwin == 0) return;
  spin_until(st, &st->p2p_arrive, (st->p2p_gen + 1u) * q.world);
}

// Step 3 (1 thread, after the owner's finalize): signal completion to every rank, count the
// exchange.
__global__ void k_p2p_finish(const QueryDev q) {
  DevState* st = q.state;
  long long k_lo;
  uint32_t nwin;
  close_window(q, k_lo, nwin);
  if (nwin == 0) return;
  st->p2p_gen += 1u;
  signal_all(q, 1);
}

// Device-side watermark exchange (one thread; replaces the host-issued all-reduce): fold this
// rank's watermark / first ts into every rank's slot of this batch, signal arrival, wait for
// world arrivals, adopt the global values, and re-arm the slot for batch b + 2.  A rank can
// run at most one batch ahead of the slowest (its next fold waits on everyone's arrival of
// the current batch), so two slots suffice.
__global__ void k_wm_exchange(const QueryDev q) {
  DevState* st = q.state;
  const unsigned int gen = st->wmx_gen, slot = gen & 1u;
  const unsigned long long wm = st->wm, tsmin = st->ts_min;
  for (uint32_t r = 0; r < q.world; r++) {
    DevState* ps = q.peers[r].state;
    atomicMax_system(&ps->wmx_max[slot], wm);
    atomicMin_system(&ps->wmx_min[slot], tsmin);
  }
  __threadfence_system();
  for (uint32_t r = 0; r < q.world; r++) atomicAdd_system(&q.peers[r].state->wmx_arrive, 1u);
  spin_until(st, &st->wmx_arrive, (gen + 1u) * q.world);
  st->wm = *(volatile unsigned long long*)&st->wmx_max[slot];
  st->ts_min = *(volatile unsigned long long*)&st->wmx_min[slot];
  // re-arm my slot for batch gen + 2: a peer folds into it only after every rank (me included)
  // has arrived for batch gen + 1, which I do after this
  st->wmx_max[slot] = 0;
  st->wmx_min[slot] = 0xFFFFFFFFull;
  st->wmx_gen = gen + 1u;
  __threadfence_system();
}

__device__ __forceinline__ unsigned long long append_row(DevState* st, bool want) {
  const uint32_t act = __activemask();
  const uint32_t m = __ballot_sync(act, want);
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long base = 0;
  const int leader = m ? __ffs(m) - 1 : 0;
  if (m && (int)lane == leader) base = atomicAdd(&st->rows, (unsigned long long)__popc(m));
  base = __shfl_sync(act, base, leader);
  return base + __popc(m & ((1u << lane) - 1u));
}

// Merged accumulators -> final rows (AVG, HAVING) for LR2 / CM2; zeroes what it reads.
__global__ void __launch_bounds__(kThreads) k_finalize(const QueryDev q, long long k_lo, uint32_t nwin) {
  DevState* st = q.state;
  if (nwin == 0) close_window(q, k_lo, nwin);
  const uint32_t K = q.kind == kCM2S ? min(st->n_keys, q.K) : q.K;
  const bool nvls = q.mc_sum != nullptr && dense_kind(q);
  if (nvls) fence_alias();                     // replica reads after the switch reductions
  lms_agg_row* rows = reinterpret_cast<lms_agg_row*>(q.rows);
  const unsigned long long total = (unsigned long long)nwin * K;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long iters = (total + stride - 1) / stride;
  for (unsigned long long it = 0; it < iters; it++) {
    const unsigned long long i = it * stride + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    unsigned long long s = 0, c = 0;
    uint32_t w = 0, key = 0;
    if (i < total) {
      w = (uint32_t)(i / K);
      key = (uint32_t)(i - (unsigned long long)w * K);
      const size_t g = (size_t)w * q.K + key;
      if (nvls) {
        // every replica holds every key: the key's owner emits it and zeroes it everywhere
        if ((uint32_t)(fmix64((unsigned long long)key) % q.world) == q.rank) {
          s = q.macc_sum[g];
          c = q.macc_cnt[g];
          if (c) { mc_store(q.mc_sum + g, 0ull); mc_store(q.mc_cnt + g, 0ull); }
        }
      } else {
        s = q.macc_sum[g];
        c = q.macc_cnt[g];
        if (c) { q.macc_sum[g] = 0; q.macc_cnt[g] = 0; }
      }
    }
    bool want = c > 0;
    double sum, avg;
    if (q.kind == kLR2S) {
      sum = (double)s;
      avg = want ? sum / (double)c : 0.0;
      want = want && (avg < 40.0);                             // HAVING (avgSpeed < 40.0)
    } else {
      sum = (double)s / 1e6;
      avg = want ? sum / (double)c : 0.0;
    }
    const unsigned long long pos = append_row(st, want);
    if (want) {
      if (pos < q.row_cap) {
        lms_agg_row r;
        const long long k = k_lo + (long long)w;
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
  }
}

// CM1: one CTA per instance; ORDER BY SUM(cpu) ascending, ties by category (reading R9).
__global__ void __launch_bounds__(32) k_finalize_cm1(const QueryDev q, long long k_lo, uint32_t nwin) {
  DevState* st = q.state;
  if (nwin == 0) close_window(q, k_lo, nwin);
  const uint32_t w = blockIdx.x, c = threadIdx.x;
  if (w >= nwin) return;
  const bool nvls = q.mc_sum != nullptr;
  if (nvls) {
    // every replica holds every instance: the instance's owner (k mod world) ranks it
    const long long m = (k_lo + (long long)w) % (long long)q.world;
    if ((uint32_t)(m < 0 ? m + q.world : m) != q.rank) return;
    fence_alias();
  }
  __shared__ unsigned long long s_sum[10], s_cnt[10];
  if (c < 10) {
    const size_t g = (size_t)w * q.K + c;
    s_sum[c] = q.macc_sum[g];
    s_cnt[c] = q.macc_cnt[g];
    if (nvls) { mc_store(q.mc_sum + g, 0ull); mc_store(q.mc_cnt + g, 0ull); }
    else { q.macc_sum[g] = 0; q.macc_cnt[g] = 0; }
  }
  __syncwarp();
  const bool want = c < 10 && s_cnt[c] > 0;
  uint32_t rank = 0;
  if (want)
    for (uint32_t j = 0; j < 10; j++)
      if (s_cnt[j] > 0 && (s_sum[j] < s_sum[c] || (s_sum[j] == s_sum[c] && j < c))) rank++;
  const unsigned long long pos = append_row(st, want);
  if (want) {
    lms_agg_row* rows = reinterpret_cast<lms_agg_row*>(q.rows);
    if (pos < q.row_cap) {
      lms_agg_row r;
      const long long k = k_lo + (long long)w;
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

int sm_count() {
  static int nsm = -1;
  if (nsm < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  return nsm;
}

}  // namespace

// Load every kernel of this file now (CUDA 12 loads kernels lazily, at first launch, and a
// lazy load waits for the device: a first launch behind a running spin-wait kernel of another
// handle — the multi-GPU device barriers on a shared GPU — would wait for that spin to time
// out).  Called once per process from lms_query_create.
void preload_dist_kernels() {
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k_bucket_count);
  cudaFuncGetAttributes(&fa, k_bucket_scatter);
  cudaFuncGetAttributes(&fa, k_merge);
  cudaFuncGetAttributes(&fa, k_finalize);
  cudaFuncGetAttributes(&fa, k_finalize_cm1);
  cudaFuncGetAttributes(&fa, k_p2p_push);
  cudaFuncGetAttributes(&fa, k_p2p_push_async);
  cudaFuncGetAttributes(&fa, k_p2p_wait_arrive);
  cudaFuncGetAttributes(&fa, k_p2p_finish);
  cudaFuncGetAttributes(&fa, k_wm_exchange);
}

cudaError_t launch_bucket(const QueryDev& q, cudaStream_t st) {
  k_bucket_count<<<sm_count(), kThreads, 0, st>>>(q);
  k_bucket_scatter<<<sm_count(), kThreads, 0, st>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_p2p_push(const QueryDev& q, long long k_lo, uint32_t nwin, cudaStream_t st) {
  k_p2p_push<<<sm_count(), kThreads, 0, st>>>(q, k_lo, nwin);
  return cudaGetLastError();
}

cudaError_t launch_wm_exchange(const QueryDev& q, cudaStream_t st) {
  k_wm_exchange<<<1, 1, 0, st>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_p2p_exchange_async(const QueryDev& q, cudaStream_t st) {
  k_p2p_push_async<<<sm_count(), kThreads, 0, st>>>(q);
  k_p2p_wait_arrive<<<1, 32, 0, st>>>(q);
  if (q.kind == kCM1S || q.kind == kCM1T) k_finalize_cm1<<<q.Wmerge, 32, 0, st>>>(q, 0, 0u);
  else k_finalize<<<sm_count(), kThreads, 0, st>>>(q, 0, 0u);
  k_p2p_finish<<<1, 32, 0, st>>>(q);
  return cudaGetLastError();
}

cudaError_t launch_merge_rows(const QueryDev& q, const void* rows, unsigned long long n, long long k_lo,
                              uint32_t nwin, cudaStream_t st) {
  k_merge<<<sm_count(), kThreads, 0, st>>>(q, static_cast<const lms_agg_row*>(rows), n, k_lo, nwin);
  return cudaGetLastError();
}

cudaError_t launch_merge(const QueryDev& q, const void* rows, unsigned long long n, long long k_lo,
                         uint32_t nwin, cudaStream_t st) {
  if (n) k_merge<<<sm_count(), kThreads, 0, st>>>(q, static_cast<const lms_agg_row*>(rows), n, k_lo, nwin);
  if (q.kind == kCM1S || q.kind == kCM1T) k_finalize_cm1<<<nwin, 32, 0, st>>>(q, k_lo, nwin);
  else k_finalize<<<sm_count(), kThreads, 0, st>>>(q, k_lo, nwin);
  return cudaGetLastError();
}

}  // namespace lms
