// liblmstream: C ABI (include/lmstream.h) over the B200 micro-batch pipeline.
//
// Host responsibilities (§III): dataset ingest (Alg. 1 "newFiles"), admission
// (Alg. 1 / Eq. 6, CG(dN), OS(tN)), device-preference labels (Alg. 2, Eq. 7-9, report-only:
// execution is always the GPU path), Eq. 4 / Eq. 5 metrics, Eq. 10 online InfPT.  Device
// work per micro-batch: one aggregate-pass launch per <= 16 input segments, one close
// launch (+ LR1 evict), one 88 B report copy; rows are copied after completion.
#include <cuda.h>            // driver types only: functions come from cudaGetDriverEntryPoint
#include <cuda_runtime.h>

#include <array>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <algorithm>
#include <limits>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/lmstream.h"
#include "device.h"
#include "host_control.h"

using namespace lms;

namespace {

thread_local std::string g_err;

lms_status fail(lms_status s, const std::string& m) {
  g_err = m;
  return s;
}

#define CUDA_TRY(x)                                                                       \
  do {                                                                                    \
    cudaError_t e_ = (x);                                                                 \
    if (e_ != cudaSuccess) return fail(LMS_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

double now_host() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

struct Pending {
  uint64_t id;
  double ingest;
  uint64_t nbytes;
  const uint8_t* dptr;   // borrowed device buffer, or nullptr (host-pushed, in d_in)
  double h2d_s;
};

bool table_iv(int kind, uint32_t& R, uint32_t& S) {
  switch (kind) {   // Table IV
    case kLR1S: R = 30; S = 5; return true;
    case kLR1T: R = 30; S = 30; return true;
    case kLR2S: R = 30; S = 10; return true;
    case kCM1S: R = 60; S = 10; return true;
    case kCM1T: R = 60; S = 60; return true;
    case kCM2S: R = 60; S = 5; return true;
    default: return false;
  }
}
bool is_lr(int k) { return k == kLR1S || k == kLR1T || k == kLR2S; }
bool is_tumbling(int k) { return k == kLR1T || k == kCM1T; }
bool is_lr1(int k) { return k == kLR1S || k == kLR1T; }

uint64_t next_pow2(uint64_t v) {
  uint64_t p = 1;
  while (p < v) p <<= 1;
  return p;
}

// FIFO of result rows drained by lms_read_* (contiguous storage + read offset).
template <typename T>
struct RowFifo {
  // Result rows waiting for lms_read_*: pinned host memory, so the device rows are copied by
  // DMA straight into the FIFO's tail (one D2H, one copy into the caller's array).
  T* buf = nullptr;
  uint64_t cap = 0, head = 0, tail = 0;
  ~RowFifo() { if (buf) cudaFreeHost(buf); }
  cudaError_t reserve(uint64_t extra) {
    if (tail + extra <= cap) return cudaSuccess;
    const uint64_t live = tail - head;
    if (live + extra <= cap && buf) {            // compact in place
      std::memmove(buf, buf + head, live * sizeof(T));
    } else {
      const uint64_t ncap = std::max<uint64_t>(2 * cap, live + extra);
      T* nb = nullptr;
      cudaError_t e = cudaHostAlloc((void**)&nb, ncap * sizeof(T), cudaHostAllocDefault);
      if (e != cudaSuccess) return e;
      std::memset(static_cast<void*>(nb), 0, ncap * sizeof(T));      // touch the pages now
      if (live) std::memcpy(static_cast<void*>(nb), buf + head, live * sizeof(T));
      if (buf) cudaFreeHost(buf);
      buf = nb;
      cap = ncap;
    }
    head = 0;
    tail = live;
    return cudaSuccess;
  }
  T* tail_ptr() { return buf + tail; }
  void commit(uint64_t n) { tail += n; }
  uint64_t size() const { return tail - head; }
  uint64_t read(T* dst, uint64_t n_max) {
    const uint64_t n = std::min<uint64_t>(n_max, size());
    if (n) std::memcpy(static_cast<void*>(dst), buf + head, n * sizeof(T));
    head += n;
    if (head == tail) head = tail = 0;
    return n;
  }
};

}  // namespace

struct lms_query {
  lms_config cfg{};
  int kind = 0;
  uint32_t R = 0, S = 0, ppw = 0, P = 0;
  cudaStream_t stream = nullptr, copy_stream = nullptr;
  QueryDev qd{};
  std::vector<void*> dallocs;
  uint8_t* d_in[2] = {nullptr, nullptr};
  uint64_t in_cap = 0, in_used[2] = {0, 0};
  int in_cur = 0;
  // lms_push_pinned: asynchronous H2D into staging buffer b on the copy stream, bracketed by
  // these events; the batch that consumes buffer b waits for ev_h2d_end[b] on the device
  cudaEvent_t ev_h2d_start[2] = {nullptr, nullptr}, ev_h2d_end[2] = {nullptr, nullptr};
  bool h2d_pending[2] = {false, false};
  std::vector<Pending> pending;
  uint64_t next_ds_id = 0;
  double last_ingest = -std::numeric_limits<double>::infinity();
  // Eq. 4 / Eq. 5 / Eq. 10 history
  std::vector<double> maxlat_hist;
  double cum_bytes = 0, cum_proc = 0;
  double next_trigger = 0;
  double infpt = 150e3;
  std::deque<std::array<double, 3>> reg_hist;
  RefitWorker refit;               // Eq. 10 refit off the batch path
  Dag dag;
  // in-flight batches: slot `cur_slot` holds the newest batch (in_flight), and with
  // LMS_FLAG_PIPELINE up to kPipeDepth - 1 older slots hold earlier, still running batches
  // (parked, oldest = cur_slot - n_parked), so the host prepares and launches batch i+1 while
  // the GPU runs batches i, i-1: a host stall shorter than two batches does not idle the GPU
  struct Flight {
    lms_batch_record cur{};
    int in_buf = 0;
    bool h2d_async = false;            // its staging buffer was filled by lms_push_pinned
    bool flush = false;
    cudaEvent_t ev_admit = nullptr, ev_start = nullptr, ev_agg = nullptr, ev_close = nullptr;
    // the batch's device-time start: ev_start only when a wait on an asynchronous H2D sits
    // between admission and the kernels, otherwise the admission event itself (one event record
    // fewer per batch); ev_close also marks the batch's end (nothing is enqueued after it)
    cudaEvent_t start() const { return start_is_admit ? ev_admit : ev_start; }
    bool start_is_admit = false;
    BatchReport* h_report = nullptr;   // mapped pinned
    BatchReport* d_report = nullptr;
    void* d_rows = nullptr;            // result rows of this batch
  };
  static constexpr int kPipeDepth = 3;
  Flight fl[kPipeDepth];
  int cur_slot = 0;
  bool pipeline = false;
  int n_parked = 0;
  bool in_flight = false;
  bool awaiting_close = false;     // multi-GPU: aggregate pass launched, close not yet
  bool p2p_async_pending = false;  // fused exchange enqueued behind the close (lms_p2p_collect)
  bool device_wm = false;          // multi-GPU: watermark exchanged by a kernel (lms_p2p_device_watermark)
  BatchReport last_report{};
  Flight& F() { return fl[cur_slot]; }
  std::vector<lms_batch_record> records;
  RowFifo<lms_agg_row> agg_rows;
  RowFifo<lms_lr1_row> lr1_rows;
  unsigned long long* h_count = nullptr;   // pinned 8 B (merged row count)
  std::vector<PeerView> peers_h;           // fused exchange: every rank's owner state
  std::vector<void*> ipc_opened;           // peer buffers opened with cudaIpcOpenMemHandle
  uint64_t launches = 0;
  double last_batch_s = 0, last_agg_s = 0, last_close_s = 0;
  // completion status of a batch that lms_push had to complete itself (pipelined handle whose
  // staging buffer still fed the parked batch): reported by the next lms_sync / lms_poll /
  // lms_force_batch instead of being dropped
  lms_status deferred_status = LMS_OK;
  std::string deferred_msg;
  bool rehash_pending = false;     // a batch report asked for the grid-wide dictionary rebuild
  bool poisoned = false;           // a fused-exchange barrier timed out: ranks may disagree on the
                                   // window state, so every later batch call fails (LMS_ESTATE)
  // single-handle multi-device driver (cfg.num_gpus > 1): one sub-handle (rank g of G) per device;
  // this handle keeps the host side (pending datasets, Alg. 1 / Eq. 4-6 / Eq. 10 history, batch
  // records, row FIFOs) of the whole, row-partitioned micro-batch
  std::vector<lms_query*> subs;
  std::vector<cudaEvent_t> g_end;          // per sub: after the batch's last kernel (its stream)
  std::vector<uint32_t*> g_lr1_w;          // LR1: per sub, the device-summed window counts
  lms_batch_record g_cur{};
  bool g_in_flight = false;
  // NVLS merge tables (group handles of dense kinds): one multicast object, one physical
  // replica per distinct device, their unicast mappings and the multicast mapping
  struct Nvls {
    bool active = false;
    CUmemGenericAllocationHandle mc = 0;
    std::vector<CUmemGenericAllocationHandle> phys;
    std::vector<CUdeviceptr> uc;
    std::vector<int> dev;
    CUdeviceptr mcva = 0;
    size_t size = 0;
  } nvls;
  void nvls_release();

  ~lms_query() {
    nvls_release();
    for (size_t g = 0; g < subs.size(); g++) {
      if (g < g_end.size() && g_end[g]) { cudaSetDevice(subs[g]->cfg.device); cudaEventDestroy(g_end[g]); }
      delete subs[g];
    }
    cudaSetDevice(cfg.device);
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    for (void* p : dallocs) cudaFree(p);
    for (cudaEvent_t e : {ev_h2d_start[0], ev_h2d_start[1], ev_h2d_end[0], ev_h2d_end[1]})
      if (e) cudaEventDestroy(e);
    for (Flight& f : fl) {
      if (f.h_report) cudaFreeHost(f.h_report);
      for (cudaEvent_t e : {f.ev_admit, f.ev_start, f.ev_agg, f.ev_close})
        if (e) cudaEventDestroy(e);
    }
    if (h_count) cudaFreeHost(h_count);
    if (stream) cudaStreamDestroy(stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
  }

  template <typename T>
  lms_status dalloc(T** p, size_t n_elems, int fill_byte) {
    void* v = nullptr;
    const size_t bytes = std::max<size_t>(n_elems * sizeof(T), 16);
    cudaError_t e = cudaMalloc(&v, bytes);
    if (e != cudaSuccess) return fail(LMS_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    dallocs.push_back(v);
    e = cudaMemset(v, fill_byte, bytes);
    if (e != cudaSuccess) return fail(LMS_ECUDA, cudaGetErrorString(e));
    *p = static_cast<T*>(v);
    return LMS_OK;
  }
};

namespace {

lms_status validate_config(const lms_config* c) {
  if (!c) return fail(LMS_EINVAL, "null config");
  if (c->struct_size != sizeof(lms_config)) return fail(LMS_EINVAL, "struct_size mismatch");
  uint32_t R, S;
  if (!table_iv(c->kind, R, S)) return fail(LMS_EINVAL, "unknown query kind");
  if (c->mode < 0 || c->mode > 3) return fail(LMS_EINVAL, "unknown mode");
  if (c->mode == LMS_MODE_TRIGGER && !(c->trigger_s > 0)) return fail(LMS_EINVAL, "trigger_s must be > 0");
  if (c->mode == LMS_MODE_DEADLINE && !(c->deadline_s >= 0)) return fail(LMS_EINVAL, "deadline_s must be >= 0");
  if (c->range_s < 0 || c->slide_s < 0) return fail(LMS_EINVAL, "negative window");
  if (c->range_s != std::floor(c->range_s) || c->slide_s != std::floor(c->slide_s))
    return fail(LMS_EINVAL, "window range/slide must be whole seconds");
  if (c->num_cores < 1) return fail(LMS_EINVAL, "num_cores < 1");
  if (c->num_xways < 1 || c->num_xways > 16) return fail(LMS_EINVAL, "num_xways must be 1..16");
  if (!(c->inf_pt_bytes > 0) || !(c->base_trans_cost >= 0)) return fail(LMS_EINVAL, "bad cost constants");
  if (c->max_batch_bytes == 0 || c->max_batch_bytes > kMaxBatchTotal) return fail(LMS_EINVAL, "max_batch_bytes must be in [1, 2^37]");
  if (c->max_keys == 0 || c->max_keys > (1ull << 30)) return fail(LMS_EINVAL, "max_keys");
  if (c->max_result_rows == 0 || c->max_result_rows > (1ull << 32)) return fail(LMS_EINVAL, "max_result_rows");
  if (c->world < 1 || c->world > kMaxWorld || c->rank < 0 || c->rank >= c->world)
    return fail(LMS_EINVAL, "need 0 <= rank < world <= 64");
  if (c->world > 1 && c->mode != LMS_MODE_MANUAL)
    return fail(LMS_EINVAL, "multi-GPU handles use LMS_MODE_MANUAL (the caller forms batches in lockstep)");
  if (c->num_gpus < 1 || c->num_gpus > kMaxWorld) return fail(LMS_EINVAL, "num_gpus must be 1..64");
  if (c->num_gpus > 1 && (c->world != 1 || c->rank != 0))
    return fail(LMS_EINVAL, "num_gpus > 1 drives all devices from one handle: rank / world stay 0 / 1");
  return LMS_OK;
}

lms_status launch_close_stage(lms_query* q);

// Alg. 2 labels of a batch (report-only): Part = batch bytes / NumCores.
void plan_labels(lms_query* q, lms_batch_record& r) {
  // InfPT_i is first needed here: collect the asynchronous Eq. 10 refit started when the
  // previous batch completed (its wait is the batch's optimisation blocking, Table V)
  if (q->refit.pending()) q->refit.collect(q->infpt, r.opt_overhead_s, r.opt_block_s);
  r.inf_pt_bytes = q->infpt;
  const double t0 = now_host();
  std::vector<uint8_t> dev;
  const double part = (double)r.batch_bytes / (double)q->cfg.num_cores;
  if (part > 0 && map_device(q->dag, part, q->infpt, q->cfg.base_trans_cost, dev)) {
    for (size_t o = 0; o < dev.size(); o++) {
      if (dev[o]) { r.n_gpu_ops++; r.plan_mask |= 1u << o; }
      else r.n_cpu_ops++;
    }
  }
  r.plan_overhead_s = now_host() - t0;
}

// Alg. 1 for one poll at `now` on the handle's buffered datasets (modes LMSTREAM / DEADLINE /
// TRIGGER; MANUAL never admits here).
void alg1_decide(lms_query* q, double now, bool& admit, int32_t& reason, double& est) {
  const Mode mode = (Mode)q->cfg.mode;
  admit = false;
  reason = kBuffer;
  est = std::nan("");
  if (mode == Mode::Trigger) {
    if (now >= q->next_trigger) {                 // OS(tN): trigger instants N, 2N, ...
      q->next_trigger = (std::floor(now / q->cfg.trigger_s) + 1.0) * q->cfg.trigger_s;
      if (!q->pending.empty()) { admit = true; reason = kAdmitTrigger; }
    }
  } else if (mode == Mode::LMStream || mode == Mode::Deadline) {
    const size_t n = q->pending.size();
    std::vector<double> ing(n);
    std::vector<uint64_t> by(n);
    for (size_t j = 0; j < n; j++) { ing[j] = q->pending[j].ingest; by[j] = q->pending[j].nbytes; }
    const double thp = q->cum_proc > 0 ? q->cum_bytes / q->cum_proc : 0.0;
    const double slide = is_tumbling(q->kind) ? 0.0 : (double)q->S;   // SlideTime (Table I)
    AdmitResult ar = admit_decision(mode, slide, q->cfg.deadline_s, now, ing.data(), by.data(), n, thp,
                                    q->maxlat_hist.data(), q->maxlat_hist.size());
    admit = ar.admit;
    reason = ar.reason;
    est = ar.est;
  }
}

// Eq. 4 / Eq. 5 bookkeeping of a completed batch, and the optional Eq. 10 refit.
void account_batch(lms_query* q, lms_batch_record& r) {
  r.max_lat_s = r.max_buff_s + r.proc_s;                     // Eq. 5
  q->cum_bytes += (double)r.batch_bytes;                     // Eq. 4
  q->cum_proc += r.proc_s;
  r.avg_thput_Bps = q->cum_proc > 0 ? q->cum_bytes / q->cum_proc : 0;
  if (r.num_datasets > 0) q->maxlat_hist.push_back(r.max_lat_s);
  q->records.push_back(r);
  if ((q->cfg.flags & LMS_FLAG_ONLINE_INFPT) && r.num_datasets > 0) {
    // Eq. 10: training rows = (AvgThPut, MaxLat) -> InfPT of past batches (the
    // newest 256); test inputs = the maximum past throughput and the target latency
    // (SlideTime, Eq. 2, or the mean past MaxLat for tumbling windows, Eq. 3).  The fit runs
    // on the worker thread; plan_labels of the next batch collects it.
    q->reg_hist.push_back({r.avg_thput_Bps, r.max_lat_s, r.inf_pt_bytes});
    if (q->reg_hist.size() > 256) q->reg_hist.pop_front();
    RefitWorker::Job job;
    double tmax = 0, lsum = 0;
    for (auto& h : q->reg_hist) {
      job.thput.push_back(h[0]); job.lat.push_back(h[1]); job.infpt.push_back(h[2]);
      tmax = std::max(tmax, h[0]);
      lsum += h[1];
    }
    job.target_thput = tmax;
    job.target_lat = is_tumbling(q->kind) ? lsum / (double)q->reg_hist.size() : (double)q->S;
    q->refit.submit(std::move(job));
  }
}

lms_status launch_batch(lms_query* q, double now, int32_t reason, double est, bool flush) {
  // the slot's report / rows buffers are what this batch's kernels write
  q->qd.report = q->F().d_report;
  q->qd.rows = q->F().d_rows;
  // ---- batch composition: every pending dataset (Alg. 1 admits tmpMicroBatch whole)
  lms_batch_record& r = q->F().cur;
  r = lms_batch_record{};
  r.index = q->records.size();
  r.num_datasets = q->pending.size();
  r.admit_time_s = now;
  r.max_buff_s = 0;
  double h2d = 0;
  for (size_t j = 0; j < q->pending.size(); j++) {
    const Pending& d = q->pending[j];
    r.batch_bytes += d.nbytes;
    r.max_buff_s = (j == 0) ? (now - d.ingest) : std::max(r.max_buff_s, now - d.ingest);   // Eq. 5 Buff
    h2d += d.h2d_s;
  }
  r.h2d_s = h2d;
  r.est_max_lat_s = est;
  r.admit_reason = (uint32_t)reason;
  plan_labels(q, r);
  // ---- input segments
  std::vector<Segment> segs;
  const int buf = q->in_cur;
  if (q->in_used[buf]) segs.push_back({q->d_in[buf], q->in_used[buf]});
  for (const Pending& d : q->pending)
    if (d.dptr) segs.push_back({d.dptr, d.nbytes});
  q->pending.clear();
  q->F().in_buf = buf;
  q->F().h2d_async = q->h2d_pending[buf];
  // Proc (reading R18) runs from admission: an asynchronous H2D still in flight is part of it
  CUDA_TRY(cudaEventRecord(q->F().ev_admit, q->stream));
  q->F().start_is_admit = !q->h2d_pending[buf];
  if (q->h2d_pending[buf]) {        // asynchronous pushes: the kernels wait for their H2D
    CUDA_TRY(cudaStreamWaitEvent(q->stream, q->ev_h2d_end[buf], 0));
    q->h2d_pending[buf] = false;
    CUDA_TRY(cudaEventRecord(q->F().ev_start, q->stream));
  }
  q->in_cur ^= 1;
  q->in_used[q->in_cur] = 0;

  const bool lr = is_lr(q->kind);
  if (q->rehash_pending) {          // grid-wide dictionary rebuild asked for by an earlier batch
    CUDA_TRY(launch_dict_rehash(q->qd, q->stream));
    q->launches += 2;
    q->rehash_pending = false;
  }
  for (size_t s0 = 0; s0 < segs.size(); s0 += kMaxSegs) {
    SegTable t{};
    t.n = (int)std::min<size_t>(kMaxSegs, segs.size() - s0);
    t.tile_prefix[0] = 0;
    for (int i = 0; i < t.n; i++) {
      t.s[i] = segs[s0 + i];
      const uint64_t tiles = lr ? lr_tiles(q->qd, t.s[i].nbytes) : ((t.s[i].nbytes + kCmTile - 1) / kCmTile);
      t.tile_prefix[i + 1] = t.tile_prefix[i] + tiles;
    }
    CUDA_TRY(lr ? launch_lr_agg(q->qd, t, q->stream) : launch_cm_agg(q->qd, t, q->stream));
    q->launches++;
  }
  CUDA_TRY(cudaEventRecord(q->F().ev_agg, q->stream));
  q->F().flush = flush;
  if (q->qd.world > 1 && !q->device_wm) {   // multi-GPU: the caller all-reduces the watermark first
    q->awaiting_close = true;
    return LMS_OK;
  }
  if (q->qd.world > 1) {            // device-side watermark exchange through peer memory
    CUDA_TRY(launch_wm_exchange(q->qd, q->stream));
    q->launches++;
  }
  return launch_close_stage(q);
}

// Window close (+ LR1 eviction, + multi-GPU owner bucketing), batch report, end event.
lms_status launch_close_stage(lms_query* q) {
  CUDA_TRY(launch_close(q->qd, q->F().flush ? 1 : 0, q->stream));
  q->launches += (uint64_t)close_launches(q->qd);
  if (is_lr1(q->kind)) {
    CUDA_TRY(launch_lr1_evict(q->qd, q->stream));
    q->launches++;
  }
  if (q->qd.world > 1 && !is_lr1(q->kind)) {
    CUDA_TRY(launch_bucket(q->qd, q->stream));
    q->launches += 2;
  }
  // the batch report lives in mapped pinned memory: the close kernel writes it to the host, and
  // ev_close is the batch's end event too
  CUDA_TRY(cudaEventRecord(q->F().ev_close, q->stream));
  q->awaiting_close = false;
  q->in_flight = true;
  return LMS_OK;
}

// Complete the batch of slot f (its end event, report, rows -> host FIFO, Eq. 4/5/10).
lms_status complete_flight(lms_query* q, lms_query::Flight& f) {
  CUDA_TRY(cudaEventSynchronize(f.ev_close));
  lms_batch_record& r = f.cur;
  const BatchReport rep = *f.h_report;
  float ms_total = 0, ms_agg = 0, ms_close = 0, ms_end = 0;
  CUDA_TRY(cudaEventElapsedTime(&ms_total, f.start(), f.ev_close));
  CUDA_TRY(cudaEventElapsedTime(&ms_agg, f.start(), f.ev_agg));
  CUDA_TRY(cudaEventElapsedTime(&ms_close, f.ev_agg, f.ev_close));
  CUDA_TRY(cudaEventElapsedTime(&ms_end, f.ev_admit, f.ev_close));
  q->last_batch_s = ms_total * 1e-3;
  q->last_agg_s = ms_agg * 1e-3;
  q->last_close_s = ms_close * 1e-3;
  // result rows -> host FIFO (multi-GPU: partial rows stay on the device for lms_merge)
  q->last_report = rep;
  // (LR1 rows are final on every rank: multi-GPU LR1 probes against all-reduced counts)
  const uint64_t nrows = (q->qd.world > 1 && !is_lr1(q->kind)) ? 0 : std::min<uint64_t>(rep.rows, q->cfg.max_result_rows);
  double d2h = 0;
  if (nrows) {
    const double t0 = now_host();
    // device rows -> (DMA) -> pinned host FIFO
    const uint8_t* src = static_cast<const uint8_t*>(f.d_rows);
    // on the copy stream: the batch is complete (ev_close), and a pipelined successor may be
    // running on the compute stream — the copy must not queue behind it
    if (is_lr1(q->kind)) {
      CUDA_TRY(q->lr1_rows.reserve(nrows));
      CUDA_TRY(cudaMemcpyAsync(q->lr1_rows.tail_ptr(), src, nrows * sizeof(lms_lr1_row), cudaMemcpyDeviceToHost, q->copy_stream));
    } else {
      CUDA_TRY(q->agg_rows.reserve(nrows));
      CUDA_TRY(cudaMemcpyAsync(q->agg_rows.tail_ptr(), src, nrows * sizeof(lms_agg_row), cudaMemcpyDeviceToHost, q->copy_stream));
    }
    CUDA_TRY(cudaStreamSynchronize(q->copy_stream));
    if (is_lr1(q->kind)) q->lr1_rows.commit(nrows);
    else q->agg_rows.commit(nrows);
    d2h = now_host() - t0;
  }
  q->in_used[f.in_buf] = 0;
  if (f.h2d_async) {                 // device-timed H2D of the staging buffer (lms_push_pinned)
    float ms_h2d = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms_h2d, q->ev_h2d_start[f.in_buf], q->ev_h2d_end[f.in_buf]));
    r.h2d_s += ms_h2d * 1e-3;
    f.h2d_async = false;
  }
  if (rep.rehash_req) q->rehash_pending = true;
  r.num_records = rep.n_records;
  r.device_s = q->last_batch_s;
  r.d2h_s = d2h;
  r.proc_s = ms_end * 1e-3 + d2h;                            // Proc_i (reading R18)
  r.windows_closed = rep.windows_closed;
  r.rows_emitted = rep.rows;
  r.late_records = rep.late;
  r.bad_records = rep.bad;
  r.overflow_records = rep.overflow;
  r.watermark = rep.watermark;
  account_batch(q, r);                                       // Eq. 4 / 5 (/ 10)
  lms_status st = LMS_OK;
  if (rep.bad) st = fail(LMS_EFORMAT, "batch " + std::to_string(r.index) + ": " + std::to_string(rep.bad) +
                                          " malformed records dropped");
  if (rep.overflow || rep.row_overflow || rep.key_overflow || rep.fifo_overflow)
    st = fail(LMS_EOVERFLOW, "batch " + std::to_string(r.index) + ": capacity exceeded (pane ring, keys, rows or FIFO)");
  if (rep.vid_range)
    st = fail(LMS_EINVAL, "batch " + std::to_string(r.index) + ": vehicle id >= max_keys in dense-vehicle LR1 "
                          "(multi-GPU LR1 / LMS_FLAG_DENSE_VEHICLES): those records were rejected");
  return st;
}

// Slot of the oldest parked batch.
int oldest_parked(const lms_query* q) {
  return (q->cur_slot - q->n_parked + lms_query::kPipeDepth) % lms_query::kPipeDepth;
}

// Complete the oldest in-flight batch (the parked ones first, oldest first).
lms_status complete(lms_query* q) {
  if (q->n_parked > 0) {
    const int sl = oldest_parked(q);
    q->n_parked--;
    return complete_flight(q, q->fl[sl]);
  }
  if (!q->in_flight) return LMS_OK;
  q->in_flight = false;
  return complete_flight(q, q->F());
}

// A completion status lms_push deferred (first error wins over s).
lms_status take_deferred(lms_query* q, lms_status s) {
  if (!q->deferred_status) return s;
  const lms_status d = q->deferred_status;
  q->deferred_status = LMS_OK;
  g_err = q->deferred_msg;
  return d;
}

// Complete every in-flight batch (oldest first); the first error wins.
lms_status complete_all(lms_query* q) {
  lms_status a = LMS_OK;
  while (q->n_parked > 0 || q->in_flight) {
    const lms_status b = complete(q);
    a = a ? a : b;
  }
  return take_deferred(q, a);
}

// Pipelined handles: complete the parked batches (oldest first) until none still reads
// staging buffer `buf` (a host push is about to refill it); a format / overflow status is
// deferred to the next call.
bool parked_uses(const lms_query* q, int buf) {
  for (int i = 1; i <= q->n_parked; i++)
    if (q->fl[(q->cur_slot - i + lms_query::kPipeDepth) % lms_query::kPipeDepth].in_buf == buf) return true;
  return false;
}
lms_status release_staging(lms_query* q, int buf) {
  while (q->n_parked > 0 && parked_uses(q, buf)) {
    const lms_status c = complete(q);
    if (c && c != LMS_EFORMAT && c != LMS_EOVERFLOW) return c;
    if (c && !q->deferred_status) { q->deferred_status = c; q->deferred_msg = g_err; }
  }
  return LMS_OK;
}

// Pipelined launch (LMS_FLAG_PIPELINE): park the running batch in its slot and switch to the
// other slot, completing the batch that still occupies it first.
lms_status park_current(lms_query* q) {
  if (!q->in_flight) return LMS_OK;
  lms_status s = LMS_OK;
  if (q->n_parked == lms_query::kPipeDepth - 1) s = complete(q);   // the oldest slot is reused
  q->n_parked++;
  q->in_flight = false;
  q->cur_slot = (q->cur_slot + 1) % lms_query::kPipeDepth;
  return s;
}

}  // namespace


static lms_status push_common(lms_query* q, uint64_t nbytes, double t) {
  if (!q) return fail(LMS_EINVAL, "null query");
  if (nbytes == 0) return fail(LMS_EINVAL, "empty dataset");
  if (!(t >= q->last_ingest)) return fail(LMS_EINVAL, "ingest_time must be non-decreasing");
  if (is_lr(q->kind) && nbytes % kLrRecBytes) return fail(LMS_EINVAL, "LR dataset is not whole 70 B records");
  // one micro-batch (host-pushed + borrowed bytes) is capped at kMaxBatchTotal: the LR2 per-CTA
  // u32 partials stay exact below it (device.h)
  uint64_t pend = 0;
  for (const Pending& d : q->pending) pend += d.nbytes;
  if (nbytes > kMaxBatchTotal || pend + nbytes > kMaxBatchTotal)
    return fail(LMS_EOVERFLOW, "micro-batch would exceed 2^37 bytes (admit the buffered datasets first)");
  return LMS_OK;
}

// =====================================================================================
// Single-handle multi-device driver (cfg.num_gpus > 1; SURVEY §8(b) num_gpus / device_ids,
// §8(e) "a single process with G devices behind one lms_query handle").  The handle owns one
// sub-handle per device (rank g of G, MANUAL) and drives the multi-GPU protocol itself:
//   push        split at record boundaries (lms_split, P:417 partitions) -> each device's part
//   Alg. 1      on the whole micro-batch (total bytes; AvgThPut / MaxLat of the whole job)
//   launch      every device: aggregate pass -> device-side watermark exchange (peer memory)
//               -> close (partial rows by key owner) -> fused push into the owners'
//               accumulators -> device barrier -> owner finalize; all enqueued, no host sync
//   complete    one collect per device; the owners' rows -> this handle's FIFO; Eq. 4 / 5 with
//               Proc = the slowest device's admit -> last kernel (+ row copies)
// LR1 (self-join): watermark folded across the devices, then per closing instance every
// device's vehicle counts are summed over all devices by a peer-reading kernel and each device
// probes its own rows against the sum (no rows move); this part is host-sequenced.
namespace {

lms_status push_staged(lms_query* q, const void* src, uint64_t nbytes, double t) {
  // device (or any UVA) bytes copied into the handle's staging buffer (copy semantics)
  lms_status s = push_common(q, nbytes, t);
  if (s) return s;
  CUDA_TRY(cudaSetDevice(q->cfg.device));
  const int b = q->in_cur;
  if (q->in_used[b] + nbytes > q->in_cap) return fail(LMS_EOVERFLOW, "batch buffer full (max_batch_bytes)");
  const double t0 = now_host();
  CUDA_TRY(cudaMemcpyAsync(q->d_in[b] + q->in_used[b], src, nbytes, cudaMemcpyDefault, q->copy_stream));
  CUDA_TRY(cudaStreamSynchronize(q->copy_stream));
  q->in_used[b] += nbytes;
  q->pending.push_back({q->next_ds_id, t, nbytes, nullptr, now_host() - t0});
  q->last_ingest = t;
  q->next_ds_id++;
  return LMS_OK;
}

// ---- NVLS (NVLink SHARP) merge tables --------------------------------------------------
// Driver API functions resolved at run time (the library links the static CUDA runtime only,
// so that it loads on hosts without a driver; cudaGetDriverEntryPoint needs a device anyway).
struct DrvApi {
  bool ok = false;
  CUresult (*devAttr)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*devGet)(CUdevice*, int) = nullptr;
  CUresult (*mcCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mcGran)(size_t*, const CUmulticastObjectProp*, CUmulticastGranularity_flags) = nullptr;
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                        unsigned long long) = nullptr;
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*memCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long) = nullptr;
  CUresult (*memGran)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*addrReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
};

const DrvApi& drv() {
  static DrvApi d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult qr;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &qr) == cudaSuccess &&
             qr == cudaDriverEntryPointSuccess && *fn != nullptr;
    };
    bool ok = true;
    ok &= get("cuDeviceGetAttribute", (void**)&d.devAttr);
    ok &= get("cuDeviceGet", (void**)&d.devGet);
    ok &= get("cuMulticastCreate", (void**)&d.mcCreate);
    ok &= get("cuMulticastAddDevice", (void**)&d.mcAddDevice);
    ok &= get("cuMulticastGetGranularity", (void**)&d.mcGran);
    ok &= get("cuMulticastBindMem", (void**)&d.mcBindMem);
    ok &= get("cuMulticastUnbind", (void**)&d.mcUnbind);
    ok &= get("cuMemCreate", (void**)&d.memCreate);
    ok &= get("cuMemGetAllocationGranularity", (void**)&d.memGran);
    ok &= get("cuMemAddressReserve", (void**)&d.addrReserve);
    ok &= get("cuMemAddressFree", (void**)&d.addrFree);
    ok &= get("cuMemMap", (void**)&d.memMap);
    ok &= get("cuMemUnmap", (void**)&d.memUnmap);
    ok &= get("cuMemSetAccess", (void**)&d.memSetAccess);
    ok &= get("cuMemRelease", (void**)&d.memRelease);
    cudaGetLastError();
    d.ok = ok;
  });
  return d;
}

}  // namespace

void lms_query::nvls_release() {
  if (nvls.mc == 0 && nvls.phys.empty()) return;
  const DrvApi& d = drv();
  if (!d.ok) return;
  for (size_t i = 0; i < nvls.dev.size(); i++) cudaSetDevice(nvls.dev[i]), cudaDeviceSynchronize();
  if (nvls.mcva) { d.memUnmap(nvls.mcva, nvls.size); d.addrFree(nvls.mcva, nvls.size); }
  for (size_t i = 0; i < nvls.uc.size(); i++)
    if (nvls.uc[i]) { d.memUnmap(nvls.uc[i], nvls.size); d.addrFree(nvls.uc[i], nvls.size); }
  for (size_t i = 0; i < nvls.dev.size() && nvls.mc; i++) {
    CUdevice dv;
    if (d.devGet(&dv, nvls.dev[i]) == CUDA_SUCCESS) d.mcUnbind(nvls.mc, dv, 0, nvls.size);
  }
  for (CUmemGenericAllocationHandle h : nvls.phys) if (h) d.memRelease(h);
  if (nvls.mc) d.memRelease(nvls.mc);
  nvls = Nvls{};
}

namespace {

// Build the NVLS merge tables of a group handle (dense kinds): returns false (and leaves the
// owner-push exchange in place) when a device lacks switch multicast or any driver call fails.
bool nvls_setup(lms_query* q, const std::vector<int>& ids) {
  const DrvApi& d = drv();
  if (!d.ok) return false;
  std::vector<int> devs;
  for (int id : ids) if (std::find(devs.begin(), devs.end(), id) == devs.end()) devs.push_back(id);
  for (int id : devs) {
    CUdevice dv;
    int mc = 0;
    if (d.devGet(&dv, id) != CUDA_SUCCESS || d.devAttr(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dv) != CUDA_SUCCESS || !mc)
      return false;
  }
  const QueryDev& d0 = q->subs[0]->qd;
  const size_t half = (size_t)d0.Wmerge * d0.K * sizeof(unsigned long long);
  lms_query::Nvls& n = q->nvls;
  auto fail_out = [&]() { q->nvls_release(); cudaGetLastError(); return false; };
  // one process: no shareable handle is needed, but a driver may insist on one — try in order
  const CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                              CU_MEM_HANDLE_TYPE_FABRIC};
  CUmulticastObjectProp mp{};
  CUmemAllocationProp ap{};
  size_t gran = 0, size = 0;
  for (CUmemAllocationHandleType ht : types) {
    mp = CUmulticastObjectProp{};
    mp.numDevices = (unsigned int)devs.size();
    mp.size = 2 * half;
    mp.handleTypes = ht;
    ap = CUmemAllocationProp{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = devs[0];
    ap.requestedHandleTypes = ht;
    size_t mg = 0, pg = 0;
    if (d.mcGran(&mg, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || mg == 0 ||
        d.memGran(&pg, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || pg == 0)
      continue;
    gran = std::max(mg, pg);
    size = (mp.size + gran - 1) / gran * gran;
    mp.size = size;
    if (d.mcCreate(&n.mc, &mp) == CUDA_SUCCESS) break;
    n.mc = 0;
  }
  if (n.mc == 0) { cudaGetLastError(); return false; }
  n.size = size;
  n.dev = devs;
  for (int id : devs) {                                   // every device joins before any binds
    CUdevice dv;
    if (d.devGet(&dv, id) != CUDA_SUCCESS || d.mcAddDevice(n.mc, dv) != CUDA_SUCCESS) return fail_out();
  }
  for (int id : devs) {
    ap.location.id = id;
    CUmemGenericAllocationHandle ph = 0;
    if (d.memCreate(&ph, size, &ap, 0) != CUDA_SUCCESS) return fail_out();
    n.phys.push_back(ph);
    if (d.mcBindMem(n.mc, 0, ph, 0, size, 0) != CUDA_SUCCESS) return fail_out();
    CUdeviceptr va = 0;
    if (d.addrReserve(&va, size, gran, 0, 0) != CUDA_SUCCESS) return fail_out();
    n.uc.push_back(va);
    if (d.memMap(va, size, 0, ph, 0) != CUDA_SUCCESS) return fail_out();
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = id;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (d.memSetAccess(va, size, &acc, 1) != CUDA_SUCCESS) return fail_out();
    if (cudaSetDevice(id) != cudaSuccess || cudaMemset((void*)va, 0, size) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
      return fail_out();
  }
  if (d.addrReserve(&n.mcva, size, gran, 0, 0) != CUDA_SUCCESS) { n.mcva = 0; return fail_out(); }
  if (d.memMap(n.mcva, size, 0, n.mc, 0) != CUDA_SUCCESS) return fail_out();
  std::vector<CUmemAccessDesc> acc(devs.size());
  for (size_t i = 0; i < devs.size(); i++) {
    acc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc[i].location.id = devs[i];
    acc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  if (d.memSetAccess(n.mcva, size, acc.data(), acc.size()) != CUDA_SUCCESS) return fail_out();
  // every sub-handle: its device's replica as the merge accumulators, the multicast address
  // for the pushes / zeroing (virtual shards on one device share that device's replica)
  for (size_t g = 0; g < q->subs.size(); g++) {
    const size_t i = std::find(devs.begin(), devs.end(), ids[g]) - devs.begin();
    QueryDev& sd = q->subs[g]->qd;
    sd.macc_sum = reinterpret_cast<unsigned long long*>(n.uc[i]);
    sd.macc_cnt = reinterpret_cast<unsigned long long*>(n.uc[i] + half);
    sd.mc_sum = reinterpret_cast<unsigned long long*>(n.mcva);
    sd.mc_cnt = reinterpret_cast<unsigned long long*>(n.mcva + half);
  }
  n.active = true;
  return true;
}

lms_status group_create(const lms_config* cfg, lms_query** out) {
  lms_query* q = new (std::nothrow) lms_query();
  if (!q) return fail(LMS_ENOMEM, "host alloc");
  auto bail = [&](lms_status st) { delete q; return st; };
  q->cfg = *cfg;
  q->cfg.device_ids = nullptr;
  q->kind = cfg->kind;
  table_iv(q->kind, q->R, q->S);
  if (cfg->range_s > 0) q->R = (uint32_t)cfg->range_s;
  if (is_tumbling(q->kind)) q->S = q->R;
  else if (cfg->slide_s > 0) q->S = (uint32_t)cfg->slide_s;
  if (q->S == 0 || q->S > q->R || q->R % q->S) return bail(fail(LMS_EINVAL, "window needs 0 < S <= R, S | R"));
  q->ppw = q->R / q->S;
  q->infpt = cfg->inf_pt_bytes;
  q->next_trigger = cfg->trigger_s;
  q->dag = query_dag(q->kind);
  q->cfg.device = cfg->device_ids ? cfg->device_ids[0] : 0;
  const int G = cfg->num_gpus;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return bail(fail(LMS_ECUDA, "no CUDA device"));
  std::vector<int> ids(G);
  for (int g = 0; g < G; g++) {
    ids[g] = cfg->device_ids ? cfg->device_ids[g] : g;
    if (ids[g] < 0 || ids[g] >= ndev) return bail(fail(LMS_EINVAL, "bad device ordinal in device_ids"));
  }
  for (int a = 0; a < G; a++)          // peer access between every pair of distinct devices
    for (int b = 0; b < G; b++) {
      if (ids[a] == ids[b]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, ids[a], ids[b]);
      if (!can) return bail(fail(LMS_ECUDA, "devices without peer access (NVLink / NVSwitch needed)"));
      if (cudaSetDevice(ids[a]) != cudaSuccess) return bail(fail(LMS_ECUDA, "cudaSetDevice"));
      const cudaError_t e = cudaDeviceEnablePeerAccess(ids[b], 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return bail(fail(LMS_ECUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e)));
      cudaGetLastError();
    }
  for (int g = 0; g < G; g++) {
    lms_config c = *cfg;
    c.num_gpus = 1;
    c.device_ids = nullptr;
    c.device = ids[g];
    c.rank = g;
    c.world = G;
    c.mode = LMS_MODE_MANUAL;                      // this handle forms the batches
    c.flags &= ~(LMS_FLAG_PIPELINE | LMS_FLAG_ONLINE_INFPT);
    lms_query* sub = nullptr;
    if (lms_status st = lms_query_create(&c, &sub)) return bail(st);
    q->subs.push_back(sub);
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) return bail(fail(LMS_ECUDA, "cudaEventCreate"));
    q->g_end.push_back(e);
  }
  if (!is_lr1(q->kind)) {                          // fused exchange + device-side watermark exchange
    for (lms_query* a : q->subs)
      for (lms_query* b : q->subs)
        if (lms_status st = lms_p2p_import_local(a, b)) return bail(st);
    for (lms_query* a : q->subs)
      if (lms_status st = lms_p2p_device_watermark(a, 1)) return bail(st);
    // dense tables (LR2, CM1) with LMS_FLAG_NVLS: reduce the partials in the NVLink switch when
    // every device can join a multicast object (else the owner push stays)
    const bool dense = q->kind == kLR2S || q->kind == kCM1S || q->kind == kCM1T;
    if (dense && (cfg->flags & LMS_FLAG_NVLS)) nvls_setup(q, ids);
  } else {
    for (lms_query* a : q->subs) {
      uint32_t* w = nullptr;
      if (cudaSetDevice(a->cfg.device) != cudaSuccess) return bail(fail(LMS_ECUDA, "cudaSetDevice"));
      if (lms_status st = a->dalloc(&w, a->qd.K, 0)) return bail(st);
      q->g_lr1_w.push_back(w);
    }
  }
  const uint64_t pre = std::min<uint64_t>(cfg->max_result_rows, is_lr1(q->kind) ? (1ull << 20) : (1ull << 16));
  if (cudaSetDevice(q->cfg.device) != cudaSuccess) return bail(fail(LMS_ECUDA, "cudaSetDevice"));
  if ((is_lr1(q->kind) ? q->lr1_rows.reserve(pre) : q->agg_rows.reserve(pre)) != cudaSuccess)
    return bail(fail(LMS_ENOMEM, "pinned row FIFO"));
  *out = q;
  return LMS_OK;
}

// how: 0 host bytes (copied), 1 page-locked host bytes (asynchronous H2D), 2 device bytes
lms_status group_push(lms_query* q, const void* bytes, uint64_t nbytes, double t, uint64_t* id, int how) {
  if (nbytes == 0) return fail(LMS_EINVAL, "empty dataset");
  if (!bytes) return fail(LMS_EINVAL, "null bytes");
  if (!(t >= q->last_ingest)) return fail(LMS_EINVAL, "ingest_time must be non-decreasing");
  uint64_t pend = 0;
  for (const Pending& d : q->pending) pend += d.nbytes;
  if (nbytes > kMaxBatchTotal || pend + nbytes > kMaxBatchTotal)
    return fail(LMS_EOVERFLOW, "micro-batch would exceed 2^37 bytes (admit the buffered datasets first)");
  const uint32_t G = (uint32_t)q->subs.size();
  std::vector<uint64_t> offs(G + 1);
  if (lms_status st = lms_split(q->kind, bytes, nbytes, G, offs.data())) return st;
  int src_dev = -1;
  if (how == 2) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, bytes) != cudaSuccess || at.type != cudaMemoryTypeDevice) {
      cudaGetLastError();
      return fail(LMS_EINVAL, "not device memory");
    }
    src_dev = at.device;
  }
  for (uint32_t g = 0; g < G; g++) {
    const uint64_t m = offs[g + 1] - offs[g];
    if (!m) continue;                              // (a device may get no records of a dataset)
    const uint8_t* part = static_cast<const uint8_t*>(bytes) + offs[g];
    lms_query* sub = q->subs[g];
    lms_status st;
    if (how == 0) {
      st = lms_push(sub, part, m, t, nullptr);
    } else if (how == 1) {
      st = lms_push_pinned(sub, part, m, t, nullptr);
      if (st == LMS_EINVAL) st = lms_push(sub, part, m, t, nullptr);   // not pinned for that device
    } else if (src_dev == sub->cfg.device && !(reinterpret_cast<uintptr_t>(part) & 15u)) {
      st = lms_push_device(sub, part, m, t, nullptr);                  // borrowed in place
    } else {
      st = push_staged(sub, part, m, t);           // another device's (or unaligned) part: copy
    }
    if (st) return st;
  }
  q->pending.push_back({q->next_ds_id, t, nbytes, nullptr, 0.0});
  q->last_ingest = t;
  if (id) *id = q->next_ds_id;
  q->next_ds_id++;
  return LMS_OK;
}

lms_status group_launch(lms_query* q, double now, int32_t reason, double est, bool flush) {
  lms_batch_record& r = q->g_cur;
  r = lms_batch_record{};
  r.index = q->records.size();
  r.num_datasets = q->pending.size();
  r.admit_time_s = now;
  for (size_t j = 0; j < q->pending.size(); j++) {
    r.batch_bytes += q->pending[j].nbytes;
    r.max_buff_s = j == 0 ? now - q->pending[j].ingest : std::max(r.max_buff_s, now - q->pending[j].ingest);
  }
  r.est_max_lat_s = est;
  r.admit_reason = (uint32_t)reason;
  plan_labels(q, r);
  q->pending.clear();
  lms_status bad = LMS_OK;
  for (lms_query* sub : q->subs) {
    const lms_status st = flush ? lms_flush(sub, now) : lms_force_batch(sub, now, nullptr);
    if (st && st != LMS_EFORMAT && st != LMS_EOVERFLOW && st != LMS_EINVAL) return st;
    if (st && !bad) bad = st;
  }
  const size_t G = q->subs.size();
  if (!is_lr1(q->kind)) {
    for (lms_query* sub : q->subs)
      if (lms_status st = lms_p2p_exchange_async(sub)) return st;
  } else {
    for (lms_query* sub : q->subs) {               // aggregate passes done
      CUDA_TRY(cudaSetDevice(sub->cfg.device));
      CUDA_TRY(cudaStreamSynchronize(sub->stream));
    }
    // one global watermark / first ts (reading R7): folded across the devices' states
    unsigned long long wm = 0, tsmin = 0xFFFFFFFFull;
    for (lms_query* sub : q->subs) {
      unsigned long long v[2];
      CUDA_TRY(cudaSetDevice(sub->cfg.device));
      CUDA_TRY(cudaMemcpy(&v[0], &sub->qd.state->wm, 8, cudaMemcpyDeviceToHost));
      CUDA_TRY(cudaMemcpy(&v[1], &sub->qd.state->ts_min, 8, cudaMemcpyDeviceToHost));
      wm = std::max(wm, v[0]);
      tsmin = std::min(tsmin, v[1]);
    }
    for (lms_query* sub : q->subs) {
      CUDA_TRY(cudaSetDevice(sub->cfg.device));
      CUDA_TRY(cudaMemcpy(&sub->qd.state->wm, &wm, 8, cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(&sub->qd.state->ts_min, &tsmin, 8, cudaMemcpyHostToDevice));
    }
    int64_t k0 = 0, k1 = -1;
    if (lms_status st = lms_close_range(q->subs[0], &k0, &k1)) return st;
    std::vector<const uint32_t*> srcs(G);
    for (int64_t k = k0; k <= k1; k++) {
      for (size_t g = 0; g < G; g++) {
        void* p = nullptr;
        uint64_t n = 0;
        if (lms_status st = lms_lr1_window_counts(q->subs[g], k, &p, &n)) return st;
        srcs[g] = static_cast<const uint32_t*>(p);
      }
      for (lms_query* sub : q->subs) {             // every device's counts of instance k written
        CUDA_TRY(cudaSetDevice(sub->cfg.device));
        CUDA_TRY(cudaStreamSynchronize(sub->stream));
      }
      for (size_t g = 0; g < G; g++) {             // sum over the devices (peer reads), then probe
        lms_query* sub = q->subs[g];
        CUDA_TRY(cudaSetDevice(sub->cfg.device));
        CUDA_TRY(launch_sum_u32(q->g_lr1_w[g], srcs.data(), (uint32_t)G, sub->qd.K, sub->stream));
        QueryDev d = sub->qd;
        d.lr1_w = q->g_lr1_w[g];
        CUDA_TRY(launch_lr1_probe(d, (long long)k, sub->stream));
        sub->launches += 2;
      }
      for (lms_query* sub : q->subs) {             // before the next instance rewrites the counts
        CUDA_TRY(cudaSetDevice(sub->cfg.device));
        CUDA_TRY(cudaStreamSynchronize(sub->stream));
      }
    }
    for (lms_query* sub : q->subs)
      if (lms_status st = lms_run_close(sub)) return st;
  }
  for (size_t g = 0; g < G; g++) {
    CUDA_TRY(cudaSetDevice(q->subs[g]->cfg.device));
    CUDA_TRY(cudaEventRecord(q->g_end[g], q->subs[g]->stream));
  }
  q->g_in_flight = true;
  return bad;
}

lms_status group_complete(lms_query* q) {
  if (!q->g_in_flight) return LMS_OK;
  q->g_in_flight = false;
  lms_status first = LMS_OK;
  std::string first_msg;
  const bool lr1 = is_lr1(q->kind);
  for (lms_query* sub : q->subs) {
    const lms_status st = lr1 ? lms_sync(sub) : lms_p2p_collect(sub);
    if (st && !first) { first = st; first_msg = g_err; }
    if (st && st != LMS_EFORMAT && st != LMS_EOVERFLOW && st != LMS_EINVAL) return st;
  }
  if (!lr1) {   // a long flush: the instances beyond one merge window in host-driven passes
    int64_t k0 = 0, k1 = -1;
    if (lms_status st = lms_last_close_range(q->subs[0], &k0, &k1)) return st;
    const int64_t W = q->subs[0]->qd.Wmerge;
    for (int64_t k = k0 + W; k <= k1; k += W) {
      const uint32_t nwin = (uint32_t)std::min<int64_t>(W, k1 - k + 1);
      for (lms_query* sub : q->subs)
        if (lms_status st = lms_p2p_push(sub, k, nwin)) return st;
      for (lms_query* sub : q->subs) {
        const lms_status st = lms_p2p_finalize(sub, k, nwin);
        if (st && st != LMS_EOVERFLOW) return st;
        if (st && !first) { first = st; first_msg = g_err; }
      }
    }
  }
  lms_batch_record& r = q->g_cur;
  double proc = 0, rows_s = 0;
  const double t0 = now_host();
  for (size_t g = 0; g < q->subs.size(); g++) {
    lms_query* sub = q->subs[g];
    const lms_batch_record& sr = sub->records.back();
    r.num_records += sr.num_records;
    r.late_records += sr.late_records;
    r.bad_records += sr.bad_records;
    r.overflow_records += sr.overflow_records;
    r.device_s = std::max(r.device_s, sr.device_s);
    r.h2d_s = std::max(r.h2d_s, sr.h2d_s);
    r.d2h_s += sr.d2h_s;
    if (g == 0) { r.windows_closed = sr.windows_closed; r.watermark = sr.watermark; }
    float ms = 0;
    CUDA_TRY(cudaSetDevice(sub->cfg.device));
    CUDA_TRY(cudaEventElapsedTime(&ms, sub->F().ev_admit, q->g_end[g]));
    proc = std::max(proc, ms * 1e-3 + sr.d2h_s);
    // the device's final rows -> this handle's FIFO
    if (lr1) {
      const uint64_t n = sub->lr1_rows.size();
      CUDA_TRY(q->lr1_rows.reserve(n));
      q->lr1_rows.commit(sub->lr1_rows.read(q->lr1_rows.tail_ptr(), n));
      r.rows_emitted += n;
    } else {
      const uint64_t n = sub->agg_rows.size();
      CUDA_TRY(q->agg_rows.reserve(n));
      q->agg_rows.commit(sub->agg_rows.read(q->agg_rows.tail_ptr(), n));
      r.rows_emitted += n;
    }
  }
  rows_s = now_host() - t0;
  r.proc_s = proc + rows_s;                        // Proc_i: the slowest device (reading R18)
  account_batch(q, r);                             // Eq. 4 / 5 (/ 10) on the whole micro-batch
  if (first) g_err = first_msg;
  return first;
}

lms_status group_poll(lms_query* q, double now, int32_t* admitted, uint64_t* bidx) {
  lms_status cs = LMS_OK;
  if (q->g_in_flight) {
    for (size_t g = 0; g < q->subs.size(); g++) {
      CUDA_TRY(cudaSetDevice(q->subs[g]->cfg.device));
      const cudaError_t e = cudaEventQuery(q->g_end[g]);
      if (e == cudaErrorNotReady) return LMS_OK;   // one micro-batch in flight at a time
      if (e != cudaSuccess) return fail(LMS_ECUDA, cudaGetErrorString(e));
    }
    cs = group_complete(q);
  }
  bool admit = false;
  int32_t reason = kBuffer;
  double est = std::nan("");
  const double t0 = now_host();
  alg1_decide(q, now, admit, reason, est);
  const double admit_overhead = now_host() - t0;
  if (admit) {
    const lms_status s = group_launch(q, now, reason, est, false);
    if (s && s != LMS_EFORMAT && s != LMS_EOVERFLOW && s != LMS_EINVAL) return s;
    q->g_cur.admit_overhead_s = admit_overhead;
    if (admitted) *admitted = 1;
    if (bidx) *bidx = q->g_cur.index;
    if (s && !cs) cs = s;
  }
  return cs;
}

}  // namespace

// =====================================================================================
extern "C" {

uint32_t lms_abi_version(void) { return LMS_ABI_VERSION; }
const char* lms_last_error(void) { return g_err.c_str(); }

lms_status lms_config_init(lms_config* c, int32_t kind) {
  if (!c) return fail(LMS_EINVAL, "null config");
  uint32_t R, S;
  if (!table_iv(kind, R, S)) return fail(LMS_EINVAL, "unknown query kind");
  *c = lms_config{};
  c->struct_size = sizeof(lms_config);
  c->kind = kind;
  c->mode = LMS_MODE_LMSTREAM;
  c->device = 0;
  c->deadline_s = 0;
  c->trigger_s = 10.0;              // Baseline trigger of the final paper
  c->range_s = 0;
  c->slide_s = 0;
  c->num_cores = 12;                // executor size
  c->num_xways = 10;
  c->inf_pt_bytes = 150e3;
  c->base_trans_cost = 0.1;
  c->max_batch_bytes = is_lr1(kind) ? (256ull << 20) : (1536ull << 20);
  c->max_keys = is_lr1(kind) ? (1ull << 20) : (1ull << 16);
  c->max_result_rows = is_lr1(kind) ? (1ull << 22) : (1ull << 20);
  c->pane_slots = 0;
  c->flags = 0;
  c->rank = 0;
  c->world = 1;
  c->num_gpus = 1;
  c->device_ids = nullptr;
  return LMS_OK;
}

lms_status lms_query_create(const lms_config* cfg, lms_query** out) {
  try {
    if (!out) return fail(LMS_EINVAL, "null out");
    *out = nullptr;
    lms_status s = validate_config(cfg);
    if (s) return s;
    if (cfg->num_gpus > 1) return group_create(cfg, out);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(LMS_ECUDA, "no CUDA device");
    if (cfg->device < 0 || cfg->device >= ndev) return fail(LMS_EINVAL, "bad device ordinal");
    CUDA_TRY(cudaSetDevice(cfg->device));
    lms_query* q = new (std::nothrow) lms_query();
    if (!q) return fail(LMS_ENOMEM, "host alloc");
    q->cfg = *cfg;
    q->kind = cfg->kind;
    table_iv(q->kind, q->R, q->S);
    if (cfg->range_s > 0) q->R = (uint32_t)cfg->range_s;
    if (is_tumbling(q->kind)) q->S = q->R;                            // R19
    else if (cfg->slide_s > 0) q->S = (uint32_t)cfg->slide_s;
    if (q->S == 0 || q->S > q->R || q->R % q->S) { delete q; return fail(LMS_EINVAL, "window needs 0 < S <= R, S | R"); }
    q->ppw = q->R / q->S;
    q->P = cfg->pane_slots ? cfg->pane_slots : 2 * q->ppw + 64;
    if (q->P < q->ppw + 1 || q->ppw > 256 || q->P > 1024) {
      delete q;
      return fail(LMS_EINVAL, "need R/S <= 256 and R/S + 1 <= pane_slots <= 1024");
    }
    q->infpt = cfg->inf_pt_bytes;
    q->next_trigger = cfg->trigger_s;
    q->dag = query_dag(q->kind);
    auto bail = [&](lms_status st) { delete q; return st; };
#define Q_TRY(x) do { lms_status st_ = (x); if (st_) return bail(st_); } while (0)
#define QC_TRY(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) return bail(fail(LMS_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_))); } while (0)
    {   // every kernel loaded up front (see preload_*_kernels), once per process and device
      static std::mutex mu;
      static std::vector<int> loaded;
      std::lock_guard<std::mutex> lock(mu);
      if (std::find(loaded.begin(), loaded.end(), cfg->device) == loaded.end()) {
        preload_cm_kernels();
        preload_lr_kernels();
        preload_close_kernels();
        preload_dist_kernels();
        loaded.push_back(cfg->device);
      }
    }
    QC_TRY(cudaStreamCreateWithFlags(&q->stream, cudaStreamNonBlocking));
    QC_TRY(cudaStreamCreateWithFlags(&q->copy_stream, cudaStreamNonBlocking));
    // pipelining (two batches in flight) only for single-GPU handles
    q->pipeline = (cfg->flags & LMS_FLAG_PIPELINE) && cfg->world == 1;
    const int nslots = q->pipeline ? lms_query::kPipeDepth : 1;
    for (int sl = 0; sl < nslots; sl++) {
      lms_query::Flight& f = q->fl[sl];
      for (cudaEvent_t* e : {&f.ev_admit, &f.ev_start, &f.ev_agg, &f.ev_close}) QC_TRY(cudaEventCreate(e));
      QC_TRY(cudaHostAlloc((void**)&f.h_report, sizeof(BatchReport), cudaHostAllocMapped));
      std::memset(f.h_report, 0, sizeof(BatchReport));
      QC_TRY(cudaHostGetDevicePointer((void**)&f.d_report, f.h_report, 0));   // zero-copy report
    }
    QC_TRY(cudaHostAlloc((void**)&q->h_count, sizeof(unsigned long long), cudaHostAllocDefault));
    for (int b = 0; b < 2; b++) {
      QC_TRY(cudaEventCreate(&q->ev_h2d_start[b]));
      QC_TRY(cudaEventCreate(&q->ev_h2d_end[b]));
    }
    {   // pre-size the result FIFO (pinned, pages touched): 64 Ki aggregate rows, 1 Mi LR1 rows
        // (32 MB: an LR1 close at C2 rates emits ~0.5 M rows; growing the pinned FIFO inside a
        // batch's D2H — cudaHostAlloc + page touch — was the round-1 C2 Proc p99 outlier)
      const uint64_t pre = std::min<uint64_t>(cfg->max_result_rows, is_lr1(q->kind) ? (1ull << 20) : (1ull << 16));
      QC_TRY(is_lr1(q->kind) ? q->lr1_rows.reserve(pre) : q->agg_rows.reserve(pre));
    }

    QueryDev& d = q->qd;
    d.kind = q->kind;
    d.stripes = 1;
    d.S = q->S; d.R = q->R; d.ppw = q->ppw; d.P = q->P;
    d.div_magic = q->S > 1 ? (~0ull / q->S) + 1 : 0;
    d.num_xways = (uint32_t)cfg->num_xways;
    switch (q->kind) {
      case kLR2S: d.K = 200u * (uint32_t)cfg->num_xways; break;
      case kCM1S: case kCM1T: d.K = 10; break;
      default: d.K = (uint32_t)cfg->max_keys; break;
    }
    d.n_agg_ctas = (uint32_t)(is_lr(q->kind) ? lr_agg_ctas(d) : cm_agg_ctas(d));
    d.rank = (uint32_t)cfg->rank;
    d.world = (uint32_t)cfg->world;
    Q_TRY(q->dalloc(&d.state, 1, 0));
    d.report = q->fl[0].d_report;
    if (d.world > 1 && !is_lr1(q->kind)) {   // owner-side merge of partial rows
      lms_agg_row* send;
      Q_TRY(q->dalloc(&send, cfg->max_result_rows, 0));
      d.send_rows = send;
      d.Wmerge = q->ppw + 8;
      Q_TRY(q->dalloc(&d.macc_sum, (size_t)d.Wmerge * d.K, 0));
      Q_TRY(q->dalloc(&d.macc_cnt, (size_t)d.Wmerge * d.K, 0));
    }
    {
      const uint64_t H = next_pow2(4ull * q->P);
      d.H_mask = (uint32_t)(H - 1);
      Q_TRY(q->dalloc(&d.pane_key, H, 0xFF));
      Q_TRY(q->dalloc(&d.pane_slot, H, 0xFF));
      Q_TRY(q->dalloc(&d.slot_pane, q->P, 0xFF));
      Q_TRY(q->dalloc(&d.free_stack, q->P, 0));
      std::vector<uint32_t> fs(q->P);
      for (uint32_t i = 0; i < q->P; i++) fs[i] = q->P - 1 - i;
      QC_TRY(cudaMemcpy(d.free_stack, fs.data(), q->P * sizeof(uint32_t), cudaMemcpyHostToDevice));
    }
    if (is_lr1(q->kind)) {
      Q_TRY(q->dalloc(&d.acc_cnt32, (size_t)q->P * d.K, 0));
      if (d.world > 1 || (cfg->flags & LMS_FLAG_DENSE_VEHICLES)) d.lr1_dense = 1;   // vehicle-indexed counts
      if (d.world > 1) Q_TRY(q->dalloc(&d.lr1_w, d.K, 0));    // + the all-reduced window counts
      else Q_TRY(q->dalloc(&d.lr1_wc, (size_t)4 * d.K, 0));   // window counts of closing instances
    } else {
      // CM2: up to 16 stripes of the accumulators so that the RED.64s of a few hot jobIds spread
      // over 16 addresses (J = 100: 0.92 -> 0.34 ms per 10M records); 1.5 GB at the defaults
      // (88 slots x 64 Ki keys x 16 x 16 B, of 180 GB); stripes x K <= 2^20
      // (fewer stripes for large key spaces: the footprint, not contention, matters there)
      d.stripes = 1;
      if (q->kind == kCM2S)
        while (d.stripes < 16u && (uint64_t)d.stripes * 2u * d.K <= (1ull << 20)) d.stripes *= 2u;
      Q_TRY(q->dalloc(&d.acc_sum, (size_t)q->P * d.stripes * d.K, 0));
      Q_TRY(q->dalloc(&d.acc_cnt, (size_t)q->P * d.stripes * d.K, 0));
    }
    if (q->kind == kLR2S) {
      d.lr2_direct = std::getenv("LMS_LR2_PARTIALS") == nullptr ? 1u : 0u;   // (A/B switch)
      d.lr2_flush_tiles = 8192u;   // 8192 tiles * 512 records * speed <= 999 < 2^32
      if (const char* f = std::getenv("LMS_LR2_FLUSH_TILES"))   // test hook: exercise the flush
        d.lr2_flush_tiles = std::max(1u, std::min(8192u, (uint32_t)std::strtoul(f, nullptr, 10)));
      Q_TRY(q->dalloc(&d.part32, (size_t)d.n_agg_ctas * 4 * d.K, 0));
      Q_TRY(q->dalloc(&d.part_tag, (size_t)d.n_agg_ctas * 2, 0xFF));
    } else {
      Q_TRY(q->dalloc(&d.part_tag, (size_t)d.n_agg_ctas * 2, 0xFF));
    }
    if (q->kind == kCM2S || is_lr1(q->kind)) {
      // open addressing at load factor <= 1/4: with the keys near max_keys (LR1's default 2^20
      // vehicle slots hold ~10^6 live vehicles; CM2 with 10^6 jobIds) a quarter of the probes
      // walk past the home entry at load 1/2 — a 10M-record LR1 batch 0.37 -> 0.30 ms with the
      // 64 MB table
      const uint64_t cap = next_pow2(4 * cfg->max_keys);
      d.dict.cap_mask = cap - 1;
      d.dict.max_keys = (uint32_t)cfg->max_keys;
      Q_TRY(q->dalloc(&d.dict.keys, 2 * cap, 0xFF));   // {key, index} entries of 16 B
      Q_TRY(q->dalloc(&d.dict.free_idx, cfg->max_keys, 0));   // reclaimed-index stack
      Q_TRY(q->dalloc(&d.dict.key_by_idx, cfg->max_keys, 0));
    }
    d.row_cap = cfg->max_result_rows;
    for (int sl = 0; sl < nslots; sl++) {   // result rows, one buffer per in-flight slot
      if (is_lr1(q->kind)) {
        lms_lr1_row* rows;
        Q_TRY(q->dalloc(&rows, d.row_cap, 0));
        q->fl[sl].d_rows = rows;
      } else {
        lms_agg_row* rows;
        Q_TRY(q->dalloc(&rows, d.row_cap, 0));
        q->fl[sl].d_rows = rows;
      }
    }
    d.rows = q->fl[0].d_rows;
    if (is_lr1(q->kind)) {
      // every retained row is emitted exactly once (as an L row of its pane's instance), so
      // the FIFO never needs more room than the rows one close may emit
      d.fifo_cap = cfg->max_result_rows + 1024;
      Q_TRY(q->dalloc(&d.fifo[0], d.fifo_cap, 0));
      Q_TRY(q->dalloc(&d.fifo[1], d.fifo_cap, 0));
    }
    q->in_cap = cfg->max_batch_bytes;
    for (int b = 0; b < 2; b++) Q_TRY(q->dalloc(&q->d_in[b], q->in_cap + 4096, 0));
    DevState init{};
    init.ts_min = kEmpty32;
    init.wmx_min[0] = init.wmx_min[1] = kEmpty32;
    init.evicted_upto = -(1ll << 62);
    init.free_top = (int)q->P;
    QC_TRY(cudaMemcpy(d.state, &init, sizeof(init), cudaMemcpyHostToDevice));
    // host row FIFO pre-sized now (pinned + touched), so that no batch's result copy pays a
    // cudaHostAlloc + page touch inside its Proc (it still grows past this if not drained)
    {
      const uint64_t pre = std::min<uint64_t>(cfg->max_result_rows, 1ull << 20);
      QC_TRY(is_lr1(q->kind) ? q->lr1_rows.reserve(pre) : q->agg_rows.reserve(pre));
    }
    QC_TRY(cudaDeviceSynchronize());
#undef Q_TRY
#undef QC_TRY
    *out = q;
    return LMS_OK;
  } catch (const std::exception& e) {
    return fail(LMS_EINTERNAL, e.what());
  } catch (...) {
    return fail(LMS_EINTERNAL, "unknown exception");
  }
}

lms_status lms_query_destroy(lms_query* q) {
  try {
    delete q;
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in destroy");
  }
}


lms_status lms_push(lms_query* q, const void* bytes, uint64_t nbytes, double t, uint64_t* id) {
  try {
    if (q && !q->subs.empty()) return group_push(q, bytes, nbytes, t, id, 0);
    lms_status s = push_common(q, nbytes, t);
    if (s) return s;
    if (!bytes) return fail(LMS_EINVAL, "null bytes");
    if (!is_lr(q->kind) && static_cast<const uint8_t*>(bytes)[nbytes - 1] != '\n')
      return fail(LMS_EINVAL, "CM dataset does not end with a newline");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    // pipelined: the staging buffer may still feed a parked (earlier) batch
    if (q->n_parked > 0) {
      const lms_status c = release_staging(q, q->in_cur);
      if (c) return c;
    }
    const int b = q->in_cur;
    if (q->in_used[b] + nbytes > q->in_cap) return fail(LMS_EOVERFLOW, "batch buffer full (max_batch_bytes)");
    const double t0 = now_host();
    CUDA_TRY(cudaMemcpyAsync(q->d_in[b] + q->in_used[b], bytes, nbytes, cudaMemcpyHostToDevice, q->copy_stream));
    CUDA_TRY(cudaStreamSynchronize(q->copy_stream));
    const double h2d = now_host() - t0;
    q->in_used[b] += nbytes;
    q->pending.push_back({q->next_ds_id, t, nbytes, nullptr, h2d});
    q->last_ingest = t;
    if (id) *id = q->next_ds_id;
    q->next_ds_id++;
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in push");
  }
}

lms_status lms_push_pinned(lms_query* q, const void* bytes, uint64_t nbytes, double t, uint64_t* id) {
  try {
    if (q && !q->subs.empty()) return group_push(q, bytes, nbytes, t, id, 1);
    lms_status s = push_common(q, nbytes, t);
    if (s) return s;
    if (!bytes) return fail(LMS_EINVAL, "null bytes");
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, bytes) != cudaSuccess || at.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      return fail(LMS_EINVAL, "lms_push_pinned needs page-locked host memory (cudaHostAlloc / registered)");
    }
    if (!is_lr(q->kind) && static_cast<const uint8_t*>(bytes)[nbytes - 1] != '\n')
      return fail(LMS_EINVAL, "CM dataset does not end with a newline");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    if (q->n_parked > 0) {                                            // (see lms_push)
      const lms_status c = release_staging(q, q->in_cur);
      if (c) return c;
    }
    const int b = q->in_cur;
    if (q->in_used[b] + nbytes > q->in_cap) return fail(LMS_EOVERFLOW, "batch buffer full (max_batch_bytes)");
    if (!q->h2d_pending[b]) CUDA_TRY(cudaEventRecord(q->ev_h2d_start[b], q->copy_stream));
    CUDA_TRY(cudaMemcpyAsync(q->d_in[b] + q->in_used[b], bytes, nbytes, cudaMemcpyHostToDevice, q->copy_stream));
    CUDA_TRY(cudaEventRecord(q->ev_h2d_end[b], q->copy_stream));
    q->h2d_pending[b] = true;
    q->in_used[b] += nbytes;
    q->pending.push_back({q->next_ds_id, t, nbytes, nullptr, 0.0});   // H2D time: at completion
    q->last_ingest = t;
    if (id) *id = q->next_ds_id;
    q->next_ds_id++;
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in push_pinned");
  }
}

lms_status lms_push_device(lms_query* q, const void* dptr, uint64_t nbytes, double t, uint64_t* id) {
  try {
    if (q && !q->subs.empty()) return group_push(q, dptr, nbytes, t, id, 2);
    lms_status s = push_common(q, nbytes, t);
    if (s) return s;
    if (!dptr || (reinterpret_cast<uintptr_t>(dptr) & 15u)) return fail(LMS_EINVAL, "device pointer must be 16 B aligned");
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, dptr) != cudaSuccess || at.type != cudaMemoryTypeDevice ||
        at.device != q->cfg.device) {
      cudaGetLastError();
      return fail(LMS_EINVAL, "not device memory of the query's device");
    }
    q->pending.push_back({q->next_ds_id, t, nbytes, static_cast<const uint8_t*>(dptr), 0.0});
    q->last_ingest = t;
    if (id) *id = q->next_ds_id;
    q->next_ds_id++;
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in push_device");
  }
}

lms_status lms_poll(lms_query* q, double now, int32_t* admitted, uint64_t* bidx) {
  try {
    if (!q) return fail(LMS_EINVAL, "null query");
    if (admitted) *admitted = 0;
    if (!q->subs.empty()) return group_poll(q, now, admitted, bidx);
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    lms_status cs = LMS_OK;
    while (q->n_parked > 0) {                         // (pipelined handles polled: drain)
      const lms_status c = complete(q);
      cs = cs ? cs : c;
    }
    if (q->poisoned) return fail(LMS_ESTATE, "handle poisoned by a failed fused exchange");
    cs = take_deferred(q, cs);
    if (q->in_flight) {
      cudaError_t e = cudaEventQuery(q->F().ev_close);
      if (e == cudaErrorNotReady) return cs;        // one micro-batch in flight at a time
      if (e != cudaSuccess) return fail(LMS_ECUDA, cudaGetErrorString(e));
      lms_status c2 = complete(q);
      cs = cs ? cs : c2;
    }
    bool admit = false;
    int32_t reason = kBuffer;
    double est = std::nan("");
    const double t0 = now_host();
    alg1_decide(q, now, admit, reason, est);
    const double admit_overhead = now_host() - t0;
    if (admit) {
      lms_status s = launch_batch(q, now, reason, est, false);
      if (s) return s;
      q->F().cur.admit_overhead_s = admit_overhead;
      if (admitted) *admitted = 1;
      if (bidx) *bidx = q->F().cur.index;
    }
    return cs;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in poll");
  }
}

lms_status lms_force_batch(lms_query* q, double now, uint64_t* bidx) {
  try {
    if (!q) return fail(LMS_EINVAL, "null query");
    if (bidx) *bidx = UINT64_MAX;
    if (!q->subs.empty()) {
      if (q->g_in_flight) return fail(LMS_ESTATE, "a batch is in flight (call lms_sync)");
      if (q->pending.empty()) return LMS_OK;
      const lms_status s = group_launch(q, now, kAdmitForced, std::nan(""), false);
      if (bidx && q->g_in_flight) *bidx = q->g_cur.index;
      return s;
    }
    if (q->awaiting_close || (q->in_flight && !q->pipeline))
      return fail(LMS_ESTATE, "a batch is in flight (call lms_sync)");
    if (q->p2p_async_pending) return fail(LMS_ESTATE, "fused exchange pending (call lms_p2p_collect)");
    if (q->poisoned) return fail(LMS_ESTATE, "handle poisoned by a failed fused exchange");
    // multi-GPU ranks run their batches in lockstep: an empty rank still runs the batch
    if (q->pending.empty() && q->qd.world == 1) return LMS_OK;
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    lms_status c = take_deferred(q, park_current(q));   // pipelined: the running batch keeps its slot
    lms_status s = launch_batch(q, now, kAdmitForced, std::nan(""), false);
    if (s) return s;
    if (bidx) *bidx = q->F().cur.index;
    return c;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in force_batch");
  }
}

lms_status lms_sync(lms_query* q) {
  try {
    if (!q) return fail(LMS_EINVAL, "null query");
    if (!q->subs.empty()) return group_complete(q);
    if (q->awaiting_close) return fail(LMS_ESTATE, "multi-GPU batch: call lms_run_close first");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    return complete_all(q);
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in sync");
  }
}

lms_status lms_flush(lms_query* q, double now) {
  try {
    if (!q) return fail(LMS_EINVAL, "null query");
    if (!q->subs.empty()) {
      const lms_status s1 = group_complete(q);
      if (s1 && s1 != LMS_EFORMAT && s1 != LMS_EOVERFLOW && s1 != LMS_EINVAL) return s1;
      const lms_status s = group_launch(q, now, kAdmitFlush, std::nan(""), true);
      if (s && s != LMS_EFORMAT && s != LMS_EOVERFLOW && s != LMS_EINVAL) return s;
      const lms_status s2 = group_complete(q);
      return s1 ? s1 : (s ? s : s2);
    }
    if (q->awaiting_close) return fail(LMS_ESTATE, "multi-GPU batch: call lms_run_close first");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    lms_status s1 = complete_all(q);
    lms_status s = launch_batch(q, now, kAdmitFlush, std::nan(""), true);
    if (s) return s;
    if (q->qd.world > 1) return s1;   // the caller completes the multi-GPU protocol
    lms_status s2 = complete_all(q);
    return s2 ? s2 : s1;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in flush");
  }
}

lms_status lms_read_agg(lms_query* q, lms_agg_row* rows, uint64_t cap, uint64_t* n, uint64_t* remaining) {
  if (!q || (!rows && cap)) return fail(LMS_EINVAL, "null argument");
  if (is_lr1(q->kind)) return fail(LMS_EINVAL, "LR1 queries emit lms_lr1_row (use lms_read_lr1)");
  const uint64_t k = q->agg_rows.read(rows, cap);
  if (n) *n = k;
  if (remaining) *remaining = q->agg_rows.size();
  return LMS_OK;
}

lms_status lms_read_lr1(lms_query* q, lms_lr1_row* rows, uint64_t cap, uint64_t* n, uint64_t* remaining) {
  if (!q || (!rows && cap)) return fail(LMS_EINVAL, "null argument");
  if (!is_lr1(q->kind)) return fail(LMS_EINVAL, "not an LR1 query (use lms_read_agg)");
  const uint64_t k = q->lr1_rows.read(rows, cap);
  if (n) *n = k;
  if (remaining) *remaining = q->lr1_rows.size();
  return LMS_OK;
}

lms_status lms_num_batches(lms_query* q, uint64_t* n) {
  if (!q || !n) return fail(LMS_EINVAL, "null argument");
  *n = q->records.size();
  return LMS_OK;
}

lms_status lms_get_batch_record(lms_query* q, uint64_t i, lms_batch_record* out) {
  if (!q || !out) return fail(LMS_EINVAL, "null argument");
  if (i >= q->records.size()) return fail(LMS_EINVAL, "no such batch");
  *out = q->records[i];
  return LMS_OK;
}

lms_status lms_last_kernel_times(lms_query* q, double* batch_s, double* agg_s, double* close_s) {
  if (!q) return fail(LMS_EINVAL, "null query");
  if (!q->subs.empty()) {                          // the slowest device's
    double b = 0, a = 0, c = 0;
    for (lms_query* sub : q->subs) {
      b = std::max(b, sub->last_batch_s); a = std::max(a, sub->last_agg_s); c = std::max(c, sub->last_close_s);
    }
    if (batch_s) *batch_s = b;
    if (agg_s) *agg_s = a;
    if (close_s) *close_s = c;
    return LMS_OK;
  }
  if (batch_s) *batch_s = q->last_batch_s;
  if (agg_s) *agg_s = q->last_agg_s;
  if (close_s) *close_s = q->last_close_s;
  return LMS_OK;
}

lms_status lms_kernel_launches(lms_query* q, uint64_t* n) {
  if (!q || !n) return fail(LMS_EINVAL, "null argument");
  *n = q->launches;
  for (lms_query* sub : q->subs) *n += sub->launches;
  return LMS_OK;
}

// ------------------------------------------------------------------ multi-GPU protocol
lms_status lms_watermark_ptrs(lms_query* q, void** wm, void** tsmin, void** stream) {
  if (!q || !wm || !tsmin || !stream) return fail(LMS_EINVAL, "null argument");
  if (!q->subs.empty()) return fail(LMS_ESTATE, "a num_gpus > 1 handle runs the multi-GPU protocol itself");
  *wm = &q->qd.state->wm;
  *tsmin = &q->qd.state->ts_min;
  *stream = q->stream;
  return LMS_OK;
}

lms_status lms_run_close(lms_query* q) {
  try {
    if (!q) return fail(LMS_EINVAL, "null query");
    if (!q->awaiting_close) return fail(LMS_ESTATE, "no aggregate pass awaiting its close");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    return launch_close_stage(q);
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in run_close");
  }
}

lms_status lms_close_range(lms_query* q, int64_t* k_first, int64_t* k_last) {
  try {
    if (!q || !k_first || !k_last) return fail(LMS_EINVAL, "null argument");
    if (q->qd.world < 2) return fail(LMS_ESTATE, "not a multi-GPU handle");
    if (!q->awaiting_close) return fail(LMS_ESTATE, "no aggregate pass awaiting its close");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    CUDA_TRY(cudaStreamSynchronize(q->stream));   // the caller's watermark all-reduce is on it
    DevState s{};
    CUDA_TRY(cudaMemcpy(&s, q->qd.state, sizeof(DevState), cudaMemcpyDeviceToHost));
    // the close kernel's instance range (win_range, reading R7), computed from the same state
    *k_first = 0;
    *k_last = -1;
    if (s.wm != 0) {
      const long long W = (long long)s.wm - 1, R = q->qd.R, S = q->qd.S;
      auto fdiv = [](long long a, long long b) { long long d = a / b; return (a % b != 0 && ((a < 0) != (b < 0))) ? d - 1 : d; };
      *k_first = s.next_k_valid ? s.next_k : fdiv((long long)s.ts_min - R, S) + 1;
      *k_last = q->F().flush ? fdiv(W, S) : fdiv(W - R, S);
    }
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in close_range");
  }
}

lms_status lms_lr1_window_counts(lms_query* q, int64_t k, void** counts_dptr, uint64_t* n_counts) {
  try {
    if (!q || !counts_dptr || !n_counts) return fail(LMS_EINVAL, "null argument");
    if (!is_lr1(q->kind) || q->qd.world < 2) return fail(LMS_ESTATE, "not a multi-GPU LR1 handle");
    if (!q->awaiting_close) return fail(LMS_ESTATE, "no aggregate pass awaiting its close");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    CUDA_TRY(launch_lr1_wsum(q->qd, (long long)k, q->stream));
    q->launches++;
    *counts_dptr = q->qd.lr1_w;
    *n_counts = q->qd.K;
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in lr1_window_counts");
  }
}

lms_status lms_lr1_probe(lms_query* q, int64_t k) {
  try {
    if (!q) return fail(LMS_EINVAL, "null query");
    if (!is_lr1(q->kind) || q->qd.world < 2) return fail(LMS_ESTATE, "not a multi-GPU LR1 handle");
    if (!q->awaiting_close) return fail(LMS_ESTATE, "no aggregate pass awaiting its close");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    CUDA_TRY(launch_lr1_probe(q->qd, (long long)k, q->stream));
    q->launches++;
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in lr1_probe");
  }
}

lms_status merge_pass(lms_query* q, const void* rows, uint64_t n, long long k_lo, uint32_t nwin);

// ---- fused exchange (peer-mapped owner accumulators)
namespace {
lms_status p2p_check(lms_query* q) {
  if (!q) return fail(LMS_EINVAL, "null query");
  if (q->qd.world < 2 || is_lr1(q->kind)) return fail(LMS_ESTATE, "not a multi-GPU aggregate handle");
  return LMS_OK;
}
lms_status p2p_publish(lms_query* q) {
  if (!q->qd.peers) {
    PeerView* d = nullptr;
    if (lms_status e = q->dalloc(&d, q->qd.world, 0)) return e;
    q->qd.peers = d;
  }
  CUDA_TRY(cudaMemcpy(q->qd.peers, q->peers_h.data(), q->peers_h.size() * sizeof(PeerView), cudaMemcpyHostToDevice));
  return LMS_OK;
}
}  // namespace

static_assert(sizeof(cudaIpcMemHandle_t) == 64, "lms_p2p_handle.ipc slots are 64 B");
static_assert(sizeof(lms_p2p_handle) == 416, "lms_p2p_handle layout is part of the ABI");

lms_status lms_p2p_export(lms_query* q, lms_p2p_handle* out) {
  try {
    if (lms_status e = p2p_check(q)) return e;
    if (!out) return fail(LMS_EINVAL, "null argument");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    *out = lms_p2p_handle{};
    out->rank = q->qd.rank;
    out->world = q->qd.world;
    out->K = q->qd.K;
    out->kind = q->kind;
    out->dict_cap_mask = q->qd.dict.cap_mask;
    out->dict_max_keys = q->qd.dict.max_keys;
    void* bufs[6] = {q->qd.macc_sum, q->qd.macc_cnt, q->qd.dict.keys, q->qd.dict.free_idx, q->qd.dict.key_by_idx,
                     q->qd.state};
    for (int i = 0; i < 6; i++) {
      if (!bufs[i]) continue;                     // no dictionary for LR2 / CM1
      cudaIpcMemHandle_t h;
      CUDA_TRY(cudaIpcGetMemHandle(&h, bufs[i]));
      std::memcpy(out->ipc[i], &h, sizeof(h));
      out->present |= 1u << i;
    }
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in p2p_export");
  }
}

lms_status lms_p2p_import(lms_query* q, const lms_p2p_handle* peer) {
  try {
    if (lms_status e = p2p_check(q)) return e;
    if (!peer) return fail(LMS_EINVAL, "null argument");
    if (peer->world != q->qd.world || peer->rank >= q->qd.world || peer->K != q->qd.K || peer->kind != q->kind)
      return fail(LMS_EINVAL, "peer handle of another query shape");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    if (q->peers_h.empty()) q->peers_h.assign(q->qd.world, PeerView{});
    PeerView v{};
    if (peer->rank == q->qd.rank) {               // own rank: local pointers
      v.macc_sum = q->qd.macc_sum; v.macc_cnt = q->qd.macc_cnt; v.dict = q->qd.dict; v.state = q->qd.state;
    } else {
      void* ptr[6] = {};
      for (int i = 0; i < 6; i++) {
        if (!(peer->present & (1u << i))) continue;
        cudaIpcMemHandle_t h;
        std::memcpy(&h, peer->ipc[i], sizeof(h));
        CUDA_TRY(cudaIpcOpenMemHandle(&ptr[i], h, cudaIpcMemLazyEnablePeerAccess));
        q->ipc_opened.push_back(ptr[i]);
      }
      v.macc_sum = static_cast<unsigned long long*>(ptr[0]);
      v.macc_cnt = static_cast<unsigned long long*>(ptr[1]);
      v.dict.keys = static_cast<unsigned long long*>(ptr[2]);
      v.dict.free_idx = static_cast<uint32_t*>(ptr[3]);
      v.dict.key_by_idx = static_cast<unsigned long long*>(ptr[4]);
      v.dict.cap_mask = peer->dict_cap_mask;
      v.dict.max_keys = peer->dict_max_keys;
      v.state = static_cast<DevState*>(ptr[5]);
    }
    q->peers_h[peer->rank] = v;
    return p2p_publish(q);
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in p2p_import");
  }
}

lms_status lms_p2p_import_local(lms_query* q, lms_query* peer) {
  try {
    if (lms_status e = p2p_check(q)) return e;
    if (!peer || peer->qd.world != q->qd.world || peer->qd.K != q->qd.K || peer->kind != q->kind)
      return fail(LMS_EINVAL, "peer handle of another query shape");
    if (peer->cfg.device != q->cfg.device) {       // another device of this process: peer access
      int can = 0;
      cudaDeviceCanAccessPeer(&can, q->cfg.device, peer->cfg.device);
      if (!can) return fail(LMS_EINVAL, "in-process peers on devices without peer access");
    }
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    if (q->peers_h.empty()) q->peers_h.assign(q->qd.world, PeerView{});
    PeerView v{};
    v.macc_sum = peer->qd.macc_sum; v.macc_cnt = peer->qd.macc_cnt; v.dict = peer->qd.dict; v.state = peer->qd.state;
    q->peers_h[peer->qd.rank] = v;
    return p2p_publish(q);
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in p2p_import_local");
  }
}

lms_status lms_nvls_active(lms_query* q, int32_t* active) {
  if (!q || !active) return fail(LMS_EINVAL, "null argument");
  *active = q->nvls.active ? 1 : 0;
  return LMS_OK;
}

lms_status lms_last_close_range(lms_query* q, int64_t* k_first, int64_t* k_last) {
  if (!q || !k_first || !k_last) return fail(LMS_EINVAL, "null argument");
  if (q->in_flight || q->awaiting_close) return fail(LMS_ESTATE, "batch not complete (call lms_sync)");
  *k_first = q->last_report.close_k_first;
  *k_last = q->last_report.close_k_last;
  return LMS_OK;
}

lms_status lms_merge_window(lms_query* q, uint32_t* wmerge) {
  if (lms_status e = p2p_check(q)) return e;
  if (!wmerge) return fail(LMS_EINVAL, "null argument");
  *wmerge = q->qd.Wmerge;
  return LMS_OK;
}

lms_status lms_p2p_push(lms_query* q, int64_t k_lo, uint32_t nwin) {
  try {
    if (lms_status e = p2p_check(q)) return e;
    if (q->in_flight || q->awaiting_close) return fail(LMS_ESTATE, "batch not complete (call lms_sync)");
    if (nwin == 0 || nwin > q->qd.Wmerge) return fail(LMS_EINVAL, "nwin must be in [1, merge window]");
    for (const PeerView& v : q->peers_h)
      if (!v.macc_sum) return fail(LMS_ESTATE, "peers not imported (lms_p2p_import for every rank)");
    if (q->peers_h.size() != q->qd.world) return fail(LMS_ESTATE, "peers not imported");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    const double t0 = now_host();
    CUDA_TRY(launch_p2p_push(q->qd, (long long)k_lo, nwin, q->stream));
    q->launches++;
    CUDA_TRY(cudaStreamSynchronize(q->stream));
    if (!q->records.empty()) q->records.back().d2h_s += now_host() - t0;
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in p2p_push");
  }
}

lms_status lms_p2p_exchange_async(lms_query* q) {
  try {
    if (lms_status e = p2p_check(q)) return e;
    if (q->awaiting_close || !q->in_flight) return fail(LMS_ESTATE, "call after lms_run_close, before lms_sync");
    if (q->peers_h.size() != q->qd.world) return fail(LMS_ESTATE, "peers not imported");
    for (const PeerView& v : q->peers_h)
      if (!v.macc_sum) return fail(LMS_ESTATE, "peers not imported (lms_p2p_import for every rank)");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    CUDA_TRY(launch_p2p_exchange_async(q->qd, q->stream));
    q->launches += 4;
    q->p2p_async_pending = true;
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in p2p_exchange_async");
  }
}

lms_status lms_p2p_device_watermark(lms_query* q, int32_t enable) {
  if (lms_status e = p2p_check(q)) return e;
  if (q->in_flight || q->awaiting_close) return fail(LMS_ESTATE, "batch in flight");
  if (enable) {
    if (q->peers_h.size() != q->qd.world) return fail(LMS_ESTATE, "peers not imported");
    for (const PeerView& v : q->peers_h)
      if (!v.state) return fail(LMS_ESTATE, "peers not imported (lms_p2p_import for every rank)");
  }
  q->device_wm = enable != 0;
  return LMS_OK;
}

lms_status lms_p2p_collect(lms_query* q) {
  try {
    if (lms_status e = p2p_check(q)) return e;
    if (!q->p2p_async_pending) return fail(LMS_ESTATE, "no async exchange pending");
    if (q->poisoned) return fail(LMS_ESTATE, "handle poisoned by a failed fused exchange");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    lms_status s1 = complete_all(q);                 // batch record (the close's report)
    CUDA_TRY(cudaStreamSynchronize(q->stream));      // + the exchange kernels behind it
    q->p2p_async_pending = false;
    unsigned int err = 0;
    CUDA_TRY(cudaMemcpy(&err, &q->qd.state->p2p_err, sizeof(err), cudaMemcpyDeviceToHost));
    if (err) {
      // a bounded wait gave up: the watermark / accumulators may be partially folded and the
      // barrier generations are out of step — the handle cannot continue (fatal, not retried)
      q->poisoned = true;
      return fail(LMS_ECUDA, "fused exchange: a peer did not arrive within 20 s (handle poisoned)");
    }
    unsigned long long total = 0;
    CUDA_TRY(cudaMemcpy(&total, &q->qd.state->rows, sizeof(total), cudaMemcpyDeviceToHost));
    const uint64_t nrows = std::min<uint64_t>(total, q->cfg.max_result_rows);
    if (nrows) {
      CUDA_TRY(q->agg_rows.reserve(nrows));
      CUDA_TRY(cudaMemcpy(q->agg_rows.tail_ptr(), q->qd.rows, nrows * sizeof(lms_agg_row), cudaMemcpyDeviceToHost));
      q->agg_rows.commit(nrows);
    }
    CUDA_TRY(cudaMemset(&q->qd.state->rows, 0, sizeof(unsigned long long)));
    if (!q->records.empty()) q->records.back().rows_emitted = nrows;
    if (total > nrows) return fail(LMS_EOVERFLOW, "merged rows exceed max_result_rows");
    return s1;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in p2p_collect");
  }
}

lms_status lms_p2p_finalize(lms_query* q, int64_t k_lo, uint32_t nwin) {
  if (lms_status e = p2p_check(q)) return e;
  if (nwin == 0 || nwin > q->qd.Wmerge) return fail(LMS_EINVAL, "nwin must be in [1, merge window]");
  return merge_pass(q, nullptr, 0, (long long)k_lo, nwin);
}

lms_status lms_partials(lms_query* q, const void** rows, uint64_t* counts) {
  if (!q || !rows || !counts) return fail(LMS_EINVAL, "null argument");
  if (q->qd.world < 2 || is_lr1(q->kind)) return fail(LMS_ESTATE, "not a multi-GPU aggregate handle");
  if (q->in_flight || q->awaiting_close) return fail(LMS_ESTATE, "batch not complete (call lms_sync)");
  *rows = q->qd.send_rows;
  for (uint32_t r = 0; r < q->qd.world; r++) counts[r] = q->last_report.owner_count[r];
  return LMS_OK;
}

// Owner merge of received rows for instances [k_lo, k_lo + nwin) (rows may be null: finalize
// only, fused exchange), then final rows -> (DMA) -> pinned host FIFO.
lms_status merge_pass(lms_query* q, const void* rows, uint64_t n, long long k_lo, uint32_t nwin) {
  try {
    if (q->in_flight || q->awaiting_close) return fail(LMS_ESTATE, "batch not complete (call lms_sync)");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    const double t0 = now_host();
    CUDA_TRY(launch_merge(q->qd, rows, n, k_lo, nwin, q->stream));
    q->launches += n ? 2 : 1;
    unsigned long long* d_rows = &q->qd.state->rows;
    CUDA_TRY(cudaMemcpyAsync(q->h_count, d_rows, sizeof(unsigned long long), cudaMemcpyDeviceToHost, q->stream));
    CUDA_TRY(cudaStreamSynchronize(q->stream));
    const uint64_t total = *q->h_count;
    const uint64_t nrows = std::min<uint64_t>(total, q->cfg.max_result_rows);
    if (nrows) {
      CUDA_TRY(q->agg_rows.reserve(nrows));
      CUDA_TRY(cudaMemcpyAsync(q->agg_rows.tail_ptr(), q->qd.rows, nrows * sizeof(lms_agg_row),
                               cudaMemcpyDeviceToHost, q->stream));
      CUDA_TRY(cudaStreamSynchronize(q->stream));
      q->agg_rows.commit(nrows);
    }
    CUDA_TRY(cudaMemsetAsync(d_rows, 0, sizeof(unsigned long long), q->stream));
    if (!q->records.empty()) {
      lms_batch_record& r = q->records.back();
      r.rows_emitted += nrows;
      r.d2h_s += now_host() - t0;
    }
    if (total > nrows) return fail(LMS_EOVERFLOW, "merged rows exceed max_result_rows");
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in merge");
  }
}

// Dense exchange for the small key sets (LR2: 2000 keys, CM1: 10 categories; SURVEY §8(e):
// ReduceScatter / AllReduce of dense arrays instead of an all-to-all of partial rows).
lms_status lms_dense_partials(lms_query* q, int64_t k_lo, uint32_t nwin, void** sum_dptr, void** cnt_dptr,
                              uint64_t* n_elems) {
  try {
    if (!q || !sum_dptr || !cnt_dptr || !n_elems) return fail(LMS_EINVAL, "null argument");
    if (q->qd.world < 2 || !(q->kind == kLR2S || q->kind == kCM1S || q->kind == kCM1T))
      return fail(LMS_ESTATE, "dense exchange: multi-GPU LR2S / CM1S / CM1T handles only");
    if (q->in_flight || q->awaiting_close) return fail(LMS_ESTATE, "batch not complete (call lms_sync)");
    if (nwin == 0 || nwin > q->qd.Wmerge) return fail(LMS_EINVAL, "nwin must be in [1, merge window]");
    CUDA_TRY(cudaSetDevice(q->cfg.device));
    if (k_lo == q->last_report.close_k_first && !q->records.empty()) q->records.back().rows_emitted = 0;
    // this rank's partial rows of the instances (every owner's) -> its merge accumulators
    const uint64_t n = q->last_report.part_rows;
    if (n) {
      CUDA_TRY(launch_merge_rows(q->qd, q->qd.send_rows, n, k_lo, nwin, q->stream));
      q->launches++;
    }
    *sum_dptr = q->qd.macc_sum;
    *cnt_dptr = q->qd.macc_cnt;
    *n_elems = (uint64_t)nwin * q->qd.K;
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in dense_partials");
  }
}

lms_status lms_dense_finalize(lms_query* q, int64_t k_lo, uint32_t nwin) {
  try {
    if (!q) return fail(LMS_EINVAL, "null query");
    if (q->qd.world < 2 || !(q->kind == kLR2S || q->kind == kCM1S || q->kind == kCM1T))
      return fail(LMS_ESTATE, "dense exchange: multi-GPU LR2S / CM1S / CM1T handles only");
    if (nwin == 0 || nwin > q->qd.Wmerge) return fail(LMS_EINVAL, "nwin must be in [1, merge window]");
    if (q->qd.rank == 0) return merge_pass(q, nullptr, 0, k_lo, nwin);   // finalize (AVG, HAVING, rank)
    CUDA_TRY(cudaSetDevice(q->cfg.device));                              // the others: zero their copy
    const size_t bytes = (size_t)nwin * q->qd.K * sizeof(unsigned long long);
    CUDA_TRY(cudaMemsetAsync(q->qd.macc_sum, 0, bytes, q->stream));
    CUDA_TRY(cudaMemsetAsync(q->qd.macc_cnt, 0, bytes, q->stream));
    CUDA_TRY(cudaStreamSynchronize(q->stream));
    if (!q->records.empty()) q->records.back().rows_emitted = 0;
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in dense_finalize");
  }
}

lms_status lms_merge(lms_query* q, const void* rows, uint64_t n) {
  if (!q || (n && !rows)) return fail(LMS_EINVAL, "null argument");
  if (q->qd.world < 2 || is_lr1(q->kind)) return fail(LMS_ESTATE, "not a multi-GPU aggregate handle");
  if (q->in_flight || q->awaiting_close) return fail(LMS_ESTATE, "batch not complete (call lms_sync)");
  const BatchReport& rep = q->last_report;
  if (!q->records.empty()) q->records.back().rows_emitted = 0;
  for (long long k = rep.close_k_first; k <= rep.close_k_last; k += q->qd.Wmerge) {
    const uint32_t nwin = (uint32_t)std::min<long long>(q->qd.Wmerge, rep.close_k_last - k + 1);
    if (lms_status e = merge_pass(q, rows, n, k, nwin)) return e;
  }
  return LMS_OK;
}

// ------------------------------------------------------------------ record-boundary split
// Row partition of one dataset into `parts` contiguous ranges of whole records (SURVEY §8(e):
// the host splits each micro-batch across the GPUs; the paper splits a micro-batch into
// NumCores partitions).  LR: cut i at the 70 B multiple at or below i*n/parts.  CM:
// cut i advanced from i*n/parts to the first byte that follows a '\n' (a record is <= 256 B,
// so at most one record is scanned per cut; device buffers: that window is copied to the host).
lms_status lms_split(int32_t kind, const void* bytes, uint64_t nbytes, uint32_t parts, uint64_t* offsets) {
  try {
    uint32_t R, S;
    if (!table_iv(kind, R, S)) return fail(LMS_EINVAL, "unknown query kind");
    if (!bytes || !offsets || parts == 0 || nbytes == 0) return fail(LMS_EINVAL, "null argument or empty dataset");
    const bool lr = is_lr(kind);
    if (lr && nbytes % kLrRecBytes) return fail(LMS_EINVAL, "LR dataset is not whole 70 B records");
    cudaPointerAttributes at{};
    bool dev = false;
    if (cudaPointerGetAttributes(&at, bytes) == cudaSuccess)
      dev = at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
    cudaGetLastError();
    const uint8_t* b = static_cast<const uint8_t*>(bytes);
    auto byte_at = [&](uint64_t i, uint8_t* out) -> bool {   // (device: one small copy per window)
      if (!dev) { *out = b[i]; return true; }
      return cudaMemcpy(out, b + i, 1, cudaMemcpyDeviceToHost) == cudaSuccess;
    };
    uint8_t last = 0;
    if (!lr) {
      if (!byte_at(nbytes - 1, &last)) return fail(LMS_ECUDA, "cudaMemcpy (split)");
      if (last != '\n') return fail(LMS_EINVAL, "CM dataset does not end with a newline");
    }
    offsets[0] = 0;
    for (uint32_t i = 1; i < parts; i++) {
      uint64_t c = (uint64_t)((unsigned __int128)nbytes * i / parts);
      if (lr) {
        c -= c % kLrRecBytes;
      } else if (c > 0 && c < nbytes) {
        // first record start at or after c: the byte after a '\n' in [c-1, nbytes)
        const uint64_t lo = c - 1, hi = std::min<uint64_t>(nbytes, lo + 512);
        std::vector<uint8_t> w(hi - lo);
        if (dev) {
          if (cudaMemcpy(w.data(), b + lo, w.size(), cudaMemcpyDeviceToHost) != cudaSuccess)
            return fail(LMS_ECUDA, "cudaMemcpy (split)");
        } else {
          std::memcpy(w.data(), b + lo, w.size());
        }
        uint64_t j = 0;
        while (j < w.size() && w[j] != '\n') j++;
        if (j == w.size()) {                // a line longer than 512 B: scan on (malformed input)
          uint64_t k = hi;
          uint8_t x = 0;
          while (k < nbytes) {
            if (!byte_at(k, &x)) return fail(LMS_ECUDA, "cudaMemcpy (split)");
            if (x == '\n') break;
            k++;
          }
          c = std::min<uint64_t>(nbytes, k + 1);
        } else {
          c = lo + j + 1;
        }
      }
      offsets[i] = std::max<uint64_t>(c, offsets[i - 1]);
    }
    offsets[parts] = nbytes;
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in split");
  }
}

// ------------------------------------------------------------------ pure functions
lms_status lms_est_max_lat(const double* buff_s, const uint64_t* bytes, uint64_t n, double thp, double* out) {
  if (!buff_s || !bytes || !out || n == 0) return fail(LMS_EINVAL, "empty micro-batch");
  if (!(thp > 0)) return fail(LMS_EINVAL, "AvgThPut must be > 0");
  *out = est_max_lat(buff_s, bytes, n, thp);
  return LMS_OK;
}

lms_status lms_cpu_cost(double base, double part, double infpt, double* out) {
  if (!out || !(base > 0) || !(part > 0) || !(infpt > 0)) return fail(LMS_EINVAL, "non-positive cost input");
  *out = base * (part / infpt);   // Eq. 7
  return LMS_OK;
}
lms_status lms_gpu_cost(double base, double part, double infpt, double* out) {
  if (!out || !(base > 0) || !(part > 0) || !(infpt > 0)) return fail(LMS_EINVAL, "non-positive cost input");
  *out = base * (infpt / part);   // Eq. 8
  return LMS_OK;
}
lms_status lms_trans_cost(double btc, double part, double infpt, double* out) {
  if (!out || !(btc >= 0) || !(part > 0) || !(infpt > 0)) return fail(LMS_EINVAL, "non-positive cost input");
  *out = btc * (part / infpt);    // Eq. 9
  return LMS_OK;
}
lms_status lms_base_cost(int32_t k, double* out) {
  if (!out) return fail(LMS_EINVAL, "null out");
  const double c = base_cost(k);
  if (c < 0) return fail(LMS_EINVAL, "unknown operation kind");
  *out = c;
  return LMS_OK;
}

lms_status lms_map_device(const lms_dag* dag, double part, double infpt, double btc, uint8_t* dev_out) {
  try {
    if (!dag || !dev_out || !dag->op_kind || !dag->pred_off) return fail(LMS_EINVAL, "null argument");
    if (!(part > 0) || !(infpt > 0) || !(btc >= 0)) return fail(LMS_EINVAL, "non-positive cost input");
    Dag d;
    for (uint32_t o = 0; o < dag->n; o++) {
      if (base_cost(dag->op_kind[o]) < 0) return fail(LMS_EINVAL, "unknown operation kind");
      d.kind.push_back(dag->op_kind[o]);
      std::vector<int32_t> p;
      for (int32_t j = dag->pred_off[o]; j < dag->pred_off[o + 1]; j++) p.push_back(dag->preds[j]);
      d.preds.push_back(p);
    }
    std::vector<uint8_t> dev;
    if (!map_device(d, part, infpt, btc, dev)) return fail(LMS_EPLAN, "DAG has a cycle or not exactly one root");
    for (uint32_t o = 0; o < dag->n; o++) dev_out[o] = dev[o];
    return LMS_OK;
  } catch (...) {
    return fail(LMS_EINTERNAL, "exception in map_device");
  }
}

lms_status lms_query_dag(int32_t kind, lms_dag* out) {
  static thread_local std::vector<uint8_t> kinds[6];
  static thread_local std::vector<int32_t> offs[6], preds[6];
  uint32_t R, S;
  if (!out || !table_iv(kind, R, S)) return fail(LMS_EINVAL, "unknown query kind");
  const Dag d = query_dag(kind);
  kinds[kind] = d.kind;
  offs[kind].assign(1, 0);
  preds[kind].clear();
  for (auto& p : d.preds) {
    preds[kind].insert(preds[kind].end(), p.begin(), p.end());
    offs[kind].push_back((int32_t)preds[kind].size());
  }
  out->n = (uint32_t)d.kind.size();
  out->op_kind = kinds[kind].data();
  out->pred_off = offs[kind].data();
  out->preds = preds[kind].data();
  return LMS_OK;
}

lms_status lms_admit_decision(int32_t mode, double slide_s, double deadline_s, double now_s,
                              const double* ingest_s, const uint64_t* bytes, uint64_t n, double thp,
                              const double* maxlat_hist, uint64_t n_hist, int32_t* admit, double* est,
                              int32_t* reason) {
  if (!admit || !est || !reason || (n && (!ingest_s || !bytes)) || (n_hist && !maxlat_hist))
    return fail(LMS_EINVAL, "null argument");
  if (mode != LMS_MODE_LMSTREAM && mode != LMS_MODE_DEADLINE) return fail(LMS_EINVAL, "mode");
  const AdmitResult r = admit_decision((Mode)mode, slide_s, deadline_s, now_s, ingest_s, bytes, n, thp,
                                       maxlat_hist, n_hist);
  *admit = r.admit ? 1 : 0;
  *est = r.est;
  *reason = r.reason;
  return LMS_OK;
}

lms_status lms_infpt_fit(const double* th, const double* lat, const double* ip, uint64_t n, double* b0,
                         double* b1, double* b2) {
  if (!b0 || !b1 || !b2 || (n && (!th || !lat || !ip))) return fail(LMS_EINVAL, "null argument");
  double b[3];
  if (!infpt_fit(th, lat, ip, n, b)) return fail(LMS_EHISTORY, "insufficient or degenerate history");
  *b0 = b[0]; *b1 = b[1]; *b2 = b[2];
  return LMS_OK;
}

lms_status lms_infpt_predict(double b0, double b1, double b2, double th, double lat, double* out) {
  if (!out) return fail(LMS_EINVAL, "null out");
  const double b[3] = {b0, b1, b2};
  *out = infpt_predict(b, th, lat);
  return LMS_OK;
}

lms_status lms_percentile(const double* v, uint64_t n, double p, double* out) {
  if (!v || !out || n == 0 || !(p > 0) || p > 100) return fail(LMS_EINVAL, "bad percentile input");
  *out = percentile_nearest_rank(std::vector<double>(v, v + n), p);
  return LMS_OK;
}

}  // extern "C"
