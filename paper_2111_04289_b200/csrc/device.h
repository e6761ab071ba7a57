// Device-side data layout of the LMStream hot path and the kernel launchers.
//
// HBM layout per query (one GPU):
//   input        : raw record bytes of the micro-batch (host-pushed block, 16 B aligned,
//                  + borrowed device datasets), read once by the aggregate kernel
//   pane table   : P accumulator slots; pane index floor(ts/S) -> slot through an open-
//                  addressing table pane_key/pane_slot[H] (H >= 4P, rebuilt at eviction) and a
//                  free-slot stack, so only the number of DISTINCT live panes is bounded (not
//                  their span); a window instance k = [kS, kS+R) is panes k .. k+R/S-1 (R5, R19)
//   accumulators : acc_sum[P][K], acc_cnt[P][K] (u64, exact integer sums: LR speed, CM
//                  cpu*1e6), LR1: acc_cnt32[P][K]
//   partials     : per aggregate-CTA smem tables written as u32 (LR2) / u64 (CM1)
//                  part[C][2 slots][2][K], merged by the close kernel per key slice
//   dictionary   : open-addressing jobId / vehicle -> dense index (CM2, LR1)
//   rows         : result rows of the batch (lms_agg_row / lms_lr1_row)
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace lms {

constexpr uint32_t kEmpty32 = 0xFFFFFFFFu;
constexpr uint32_t kFail32 = 0xFFFFFFFEu;   // pane table full: the pane's records overflow
constexpr unsigned long long kEmpty64 = ~0ull;
constexpr unsigned long long kTomb64 = ~0ull - 1;   // dictionary entry of a reclaimed key (no parsed
                                                    // key reaches it: <= 19 digits < 2^64 - 2)
constexpr int kMaxSegs = 128;                          // input segments per aggregate launch
// Bytes of one micro-batch (host-pushed + borrowed segments).  Bounds the LR2 per-CTA u32
// partials: a CTA of the 296-CTA grid sees <= 2^37 / 70 / 296 < 6.7e6 records of a batch, so a
// key's speed sum (<= 100 per record) stays < 6.7e8 < 2^32 even if every record has that key.
constexpr unsigned long long kMaxBatchTotal = 1ull << 37;
constexpr int kMaxWorld = 64;                          // multi-GPU ranks
constexpr int kLrRecBytes = 70;
constexpr int kLrTileRecs = 512;                       // 256 threads x 2 records
constexpr int kLrTileBytes = kLrTileRecs * kLrRecBytes; // 35840 = 16 * 2240
constexpr int kCmWin = 4352;                           // CM warp-tile window: payload + right halo
constexpr int kCmHaloL = 16;
constexpr int kCmHaloR = 256;                          // >= max line (255) + '\n'
constexpr int kCmTile = kCmWin - kCmHaloR;             // CM warp-tile payload bytes (4096)
constexpr int kCmStage = kCmHaloL + kCmWin;
constexpr int kCmMaxLine = 255;

enum QueryKind : int32_t { kLR1S = 0, kLR1T = 1, kLR2S = 2, kCM1S = 3, kCM1T = 4, kCM2S = 5 };

// Device-resident query state (one per query).
struct DevState {
  unsigned long long wm;        // live watermark: max kept ts + 1 (0 = none)
  unsigned long long wm_prev;   // snapshot at batch start: late iff ts + 1 < wm_prev
  long long next_k;             // first window instance not yet emitted
  long long evict_upto;         // LR1: panes <= this are evicted by k_lr1_evict
  long long evicted_upto;       // LR1: evict_upto of the last eviction that ran
  unsigned int next_k_valid;
  unsigned long long ts_min;    // min kept ts of the current batch (0xFFFFFFFF = none); u64 so
                                // that multi-GPU ranks can all-reduce it as int64
  unsigned long long n_records, bad, late, overflow, rows, windows_closed;
  unsigned int row_overflow;
  unsigned int close_ticket;
  unsigned int n_keys;          // dictionary indices handed out so far (high-water mark)
  int kfree_top;                // reclaimed dictionary indices on the free stack (Dict.free_idx)
  unsigned int n_tomb;          // tombstoned dictionary entries (rehash when > capacity / 4)
  unsigned int key_overflow;
  unsigned int vid_range;       // dense-vehicle LR1: a record's VID was >= max_keys (rejected)
  unsigned int fifo_count[2];   // LR1 retained-row FIFO sizes
  unsigned int fifo_cur;        // LR1: which FIFO holds the live rows
  unsigned int fifo_overflow;
  unsigned int lr1_ticket;      // LR1 aggregate launch: CTAs done (the last advances fifo_count)
  int free_top;                 // free accumulator slots on the stack
  unsigned int pane_fail;       // a pane found no free slot (table entry marked kFail32)
  long long close_k_first, close_k_last;   // instances closed by the last close (multi-GPU)
  unsigned long long part_rows;            // partial rows of the last close (multi-GPU)
  unsigned int owner_count[kMaxWorld];     // partial rows per owner rank
  unsigned int owner_cursor[kMaxWorld];
  // fused exchange, device-side barrier: every rank adds 1 to every rank's p2p_arrive when its
  // pushes of an exchange are done, and to every rank's p2p_done when its finalize is done;
  // p2p_gen counts the exchanges that had instances to close (identical on every rank)
  unsigned int p2p_arrive, p2p_done, p2p_gen, p2p_err, p2p_ticket;
  // device-side watermark exchange (reading R7 needs one global watermark): batch b's ranks
  // fold their wm (MAX) and ts_min (MIN) into every rank's slot b % 2 and count arrivals
  unsigned long long wmx_max[2], wmx_min[2];
  unsigned int wmx_arrive, wmx_gen;
};

// Copied to the host after every batch.
struct BatchReport {
  unsigned long long n_records, bad, late, overflow, rows, windows_closed;
  long long watermark;          // -1 if none
  unsigned int n_keys, row_overflow, key_overflow, fifo_overflow, vid_range;
  unsigned int rehash_req;      // dictionary tombstones above a quarter: the host enqueues the
                                // grid-wide rebuild (launch_dict_rehash) before the next batch
  long long close_k_first, close_k_last;
  unsigned long long part_rows;
  unsigned int owner_count[kMaxWorld];
};

struct Segment {
  const uint8_t* ptr;
  unsigned long long nbytes;
};

struct SegTable {
  int n;
  Segment s[kMaxSegs];
  unsigned long long tile_prefix[kMaxSegs + 1];   // tiles before segment i
};

// Retained LR1 row (projection of the 7 output columns; vehicle via dictionary index).
struct __align__(16) Lr1Retained {
  uint32_t ts;
  uint32_t vidx;
  uint16_t speed, xway, seg;
  uint8_t lane, dir;
};

struct Dict {
  unsigned long long* keys;     // [cap][2]: entry h = {key (kEmpty64 = free), index in the low 32
                                // bits of the second word (kEmpty32 until published)} — one
                                // 16 B load resolves a key (one L2 round trip, not two)
  uint32_t* free_idx;           // [max_keys] stack of reclaimed indices (a key whose panes were all
                                // evicted frees its index; inserts take recycled indices first)
  unsigned long long* key_by_idx;  // [max_keys]
  unsigned long long cap_mask;
  uint32_t max_keys;
};

// A rank's owner-side merge state as seen from any rank (multi-GPU fused exchange): its merge
// accumulators, its key dictionary (CM2) and its DevState (dictionary counters).  Pointers are
// local for the own rank and peer-mapped (CUDA IPC over NVLink, or another handle in the same
// process) for the others.
struct PeerView {
  unsigned long long* macc_sum;
  unsigned long long* macc_cnt;
  Dict dict;
  DevState* state;
};

struct QueryDev {
  int kind;
  uint32_t S, R, ppw, P;        // slide, range (s), panes per window, ring slots
  unsigned long long div_magic; // ceil(2^64 / S) for pane = ts / S (S > 1)
  uint32_t num_xways;
  uint32_t K;                   // key-space size of the accumulators
  DevState* state;
  BatchReport* report;
  uint32_t* pane_key;           // [H] pane index or kEmpty32
  uint32_t* pane_slot;          // [H] accumulator slot (kEmpty32 until published, kFail32)
  uint32_t H_mask;              // H - 1
  uint32_t* slot_pane;          // [P] pane held by accumulator slot s (kEmpty32 = free)
  uint32_t* free_stack;         // [P]
  unsigned long long* acc_sum;  // [P][stripes][K]
  unsigned long long* acc_cnt;  // [P][stripes][K]
  uint32_t stripes;             // CM2: CTAs add into stripe blockIdx % stripes (hot keys spread
                                // over `stripes` addresses); the close sums the stripes. Else 1.
  uint32_t* acc_cnt32;          // LR1 [P][K]
  uint32_t* part32;             // LR2 [C][2][2][K]
  uint32_t lr2_direct;          // LR2: CTAs add their smem tables straight into the pane
                                // accumulators (RED.64) instead of writing part32 for the close
  uint32_t lr2_flush_tiles;     // LR2: a CTA adds its u32 tables into the accumulators every this
                                // many tiles (8192: a u32 sum cannot wrap)
  unsigned long long* part64;   // CM1 [C][2][2][K]
  unsigned long long* part_tag; // [C][2] (slot << 32 | pane), kEmpty64 = unused
  uint32_t n_agg_ctas;          // C
  Dict dict;
  void* rows;                   // lms_agg_row[] / lms_lr1_row[]
  unsigned long long row_cap;
  Lr1Retained* fifo[2];
  unsigned long long fifo_cap;
  // multi-GPU (world > 1): partial rows bucketed by owner, owner-side merge accumulators
  uint32_t rank, world;
  void* send_rows;              // lms_agg_row[row_cap], grouped by owner rank
  unsigned long long* macc_sum; // [Wmerge][K]
  unsigned long long* macc_cnt; // [Wmerge][K]
  uint32_t Wmerge;              // instances merged per merge pass
  // multi-GPU LR1: vehicles index the counts directly (VID < K), and each closing instance's
  // window counts are summed into lr1_w and all-reduced before the probe
  uint32_t lr1_dense;
  uint32_t* lr1_w;              // [K]
  uint32_t* lr1_wc;             // single GPU LR1: window counts of the first closing instances
                                // [kLr1Wc = 4][K] (k_lr1_wcache), null when not allocated
  PeerView* peers;              // [world] (fused exchange; null until lms_p2p_import)
  // NVLS (single-handle multi-device driver, dense LR2 / CM1 tables): multicast addresses of
  // the merge accumulators — every device's macc_sum / macc_cnt is its replica of one
  // multicast object, pushes reduce in the NVLink switch with multimem.red into every replica,
  // owners finalize their keys from their own replica and zero them in all replicas with
  // multimem.st.  Null: the owner-push path (remote RED.64 into the owner's accumulators).
  unsigned long long* mc_sum;
  unsigned long long* mc_cnt;
};

// Launchers (kernels_*.cu).  All asynchronous on `st`.
int lr_agg_ctas(const QueryDev& q);
uint64_t lr_tiles(const QueryDev& q, uint64_t nbytes);   // aggregate tiles of an LR segment
int cm_agg_ctas(const QueryDev& q);
size_t lr_agg_smem(const QueryDev& q);
cudaError_t launch_lr_agg(const QueryDev& q, const SegTable& segs, cudaStream_t st);
cudaError_t launch_cm_agg(const QueryDev& q, const SegTable& segs, cudaStream_t st);
cudaError_t launch_close(const QueryDev& q, int flush, cudaStream_t st);
int close_launches(const QueryDev& q);                   // kernels launch_close enqueues
cudaError_t launch_dict_rehash(const QueryDev& q, cudaStream_t st);   // 2 kernels
cudaError_t launch_lr1_evict(const QueryDev& q, cudaStream_t st);
cudaError_t launch_lr1_wsum(const QueryDev& q, long long k, cudaStream_t st);
cudaError_t launch_lr1_probe(const QueryDev& q, long long k, cudaStream_t st);
cudaError_t launch_sum_u32(uint32_t* dst, const uint32_t* const* srcs, uint32_t G, uint32_t n, cudaStream_t st);
cudaError_t launch_bucket(const QueryDev& q, cudaStream_t st);
cudaError_t launch_merge(const QueryDev& q, const void* rows, unsigned long long n, long long k_lo,
                         uint32_t nwin, cudaStream_t st);
cudaError_t launch_merge_rows(const QueryDev& q, const void* rows, unsigned long long n, long long k_lo,
                              uint32_t nwin, cudaStream_t st);   // k_merge only (no finalize)
cudaError_t launch_p2p_push(const QueryDev& q, long long k_lo, uint32_t nwin, cudaStream_t st);
cudaError_t launch_p2p_exchange_async(const QueryDev& q, cudaStream_t st);
cudaError_t launch_wm_exchange(const QueryDev& q, cudaStream_t st);
int close_ctas(const QueryDev& q);
void preload_cm_kernels();
void preload_lr_kernels();
void preload_close_kernels();
void preload_dist_kernels();

}  // namespace lms
