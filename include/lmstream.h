/*
 * lmstream.h — C ABI of the B200-native LMStream micro-batch hot path.
 *
 * LMStream (arXiv 2111.04289; /root/reference/PAPER.md, cited "P:n") runs a
 * continuous windowed streaming query as a sequence of micro-batches: datasets
 * arrive (Alg. 1 "Get all new data in the source path"), an admission
 * controller decides when the buffered datasets form a micro-batch
 * (ConstructMicroBatch, Alg. 1, Eq. 6), a planner labels every
 * operation CPU/GPU (MapDevice, Alg. 2, Eq. 7-9), the batch is
 * processed (Table IV queries) and per-batch latency metrics are
 * updated (Eq. 4, Eq. 5).  This library executes the processing
 * phase entirely in hand-written sm_100a CUDA kernels (record framing, field
 * decode, predicate + compaction, pane partial aggregation, window close); the
 * host side (admission, planning, metrics) is C++.  There is no CPU fallback.
 *
 * Conventions
 *  - extern "C", C99 types only.  Every call returns lms_status (< 0 = error)
 *    except lms_abi_version / lms_last_error.  No C++ exception crosses the ABI
 *    (caught and mapped to LMS_EINTERNAL).
 *  - lms_query is opaque and library-owned; one handle must be used by one
 *    host thread at a time; distinct handles are independent.
 *  - Times are caller-supplied seconds (virtual or wall clock).  Measured
 *    processing times (Proc) are seconds of real device time.
 *  - Output arrays are caller-owned; result rows are drained FIFO.
 *  - On error, lms_last_error() returns a thread-local message valid until the
 *    next call on the same thread.
 */
#ifndef LMSTREAM_H
#define LMSTREAM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMS_ABI_VERSION 3u

typedef struct lms_query lms_query;      /* opaque, library-owned */

typedef int32_t lms_status;
enum {
  LMS_OK = 0,
  LMS_EINVAL = -1,      /* bad argument / config              */
  LMS_ENOMEM = -2,      /* host or device allocation failed                         */
  LMS_ECUDA = -3,       /* CUDA runtime error (message in lms_last_error)           */
  LMS_ENCCL = -4,       /* collective failure (multi-GPU)                           */
  LMS_EHISTORY = -5,    /* insufficient history for Eq. 10           */
  LMS_EPLAN = -6,       /* operation DAG has a cycle / not a single root    */
  LMS_EFORMAT = -7,     /* batch contained malformed records (dropped, counted)     */
  LMS_ESTATE = -8,      /* call-order violation (e.g. force while a batch is live)  */
  LMS_EOVERFLOW = -9,   /* table / ring / result capacity exceeded                  */
  LMS_EINTERNAL = -10
};

/* Table IV queries.  S = slide, R = range, seconds.            */
typedef enum {
  LMS_LR1S = 0,   /* LR window self-join, range 30 slide 5                    */
  LMS_LR1T = 1,   /* LR window self-join, tumbling range 30                   */
  LMS_LR2S = 2,   /* LR AVG(speed) GROUP BY (highway,direction,segment)
                     HAVING avg < 40.0, range 30 slide 10                     */
  LMS_CM1S = 3,   /* CM SUM(cpu) GROUP BY category ORDER BY SUM(cpu), 60/10   */
  LMS_CM1T = 4,   /* same, tumbling range 60                                  */
  LMS_CM2S = 5    /* CM AVG(cpu) WHERE eventType == 1 GROUP BY jobId, 60/5    */
} lms_query_kind;

/* Micro-batch formation policy.                                              */
typedef enum {
  LMS_MODE_LMSTREAM = 0, /* Alg. 1: target SlideTime (sliding) / mean MaxLat (tumbling) */
  LMS_MODE_DEADLINE = 1, /* CG(dN) (P:6): Alg. 1 with SlideTime := deadline_s; d=0 -> tumbling branch */
  LMS_MODE_TRIGGER = 2,  /* OS(tN) (P:6): admit everything every trigger_s seconds */
  LMS_MODE_MANUAL = 3    /* the caller forms batches with lms_force_batch        */
} lms_mode;

/* Operation kinds of the query DAG (Table III base costs P:736-766). */
typedef enum {
  LMS_OP_SCAN = 0, LMS_OP_FILTER = 1, LMS_OP_PROJECT = 2, LMS_OP_HASHAGG = 3,
  LMS_OP_HASHJOIN = 4, LMS_OP_SORT = 5, LMS_OP_SHUFFLE = 6, LMS_OP_EXPAND = 7
} lms_op_kind;

#define LMS_DEV_CPU 0
#define LMS_DEV_GPU 1

/* Query configuration.  Call lms_config_init() first, then override fields.   */
typedef struct {
  uint32_t struct_size;      /* = sizeof(lms_config)                              */
  int32_t  kind;             /* lms_query_kind                                    */
  int32_t  mode;             /* lms_mode                                          */
  int32_t  device;           /* CUDA device ordinal                               */
  double   deadline_s;       /* CG(dN): N (>= 0)                                  */
  double   trigger_s;        /* OS(tN): N (> 0)                                   */
  double   range_s;          /* window range R; 0 -> Table IV                     */
  double   slide_s;          /* window slide S; 0 -> Table IV (tumbling: S = R)   */
  int32_t  num_cores;        /* NumCores for Eq. 7-9 partitions (Table I); default 12 */
  int32_t  num_xways;        /* LR highway domain: XWay < num_xways (1..16); default 10 */
  double   inf_pt_bytes;     /* InfPT_0 = 150e3                           */
  double   base_trans_cost;  /* baseTransCost = 0.1                       */
  uint64_t max_batch_bytes;  /* capacity of one micro-batch of host-pushed bytes  */
  uint64_t max_keys;         /* distinct-key capacity (CM2 jobIds, LR1 vehicles) live in
                                the window (evicted keys' indices are reused); defaults
                                2^16 (CM2) / 2^20 (LR1); the key dictionary holds
                                next_pow2(4 * max_keys) 16 B entries (load <= 1/4)       */
  uint64_t max_result_rows;  /* result rows one batch may emit                    */
  uint32_t pane_slots;       /* distinct live panes (accumulator slots); 0 -> 2*R/S + 64 */
  uint32_t flags;            /* LMS_FLAG_*                                        */
  int32_t  rank, world;      /* multi-GPU row partition: this handle's rank of `world`
                                (1 -> single GPU).  world > 1 (LR2S, CM1*, CM2S): every
                                rank aggregates its own rows; windows close per rank as
                                PARTIAL rows that are exchanged by key owner
                                (hash(key) % world) and merged on the owner — see
                                lms_run_close / lms_partials / lms_merge.  world > 1
                                (LR1S, LR1T): vehicle-indexed counts, window counts
                                all-reduced per closing instance — lms_lr1_window_counts. */
  int32_t  num_gpus;         /* single-handle multi-device driver: > 1 -> this
                                one handle row-partitions every micro-batch over num_gpus devices
                                of this process (rank / world must stay 0 / 1).  Pushes are split
                                at record boundaries (lms_split), Alg. 1 / CG(dN) / OS(tN) size the
                                WHOLE micro-batch once (Eq. 4/5/6 on its total bytes and its Proc =
                                the slowest device's), the partial aggregates are merged by key
                                owner through peer memory (the fused exchange, device-side
                                barriers), and rows / batch records come out of this handle as
                                from a single GPU.  Devices need peer access to each other (the
                                same ordinal may repeat: virtual shards on one GPU).  Default 1.  */
  const int32_t* device_ids; /* [num_gpus] CUDA ordinals (NULL -> 0 .. num_gpus-1); copied at
                                lms_query_create                                                */
} lms_config;

#define LMS_FLAG_ONLINE_INFPT 0x1u  /* Eq. 10 online regression of InfPT */
#define LMS_FLAG_PIPELINE     0x2u  /* single GPU: lms_force_batch may launch batch i+1 while
                                       batches i, i-1 still run (up to three batches in flight,
                                       separate report / row buffers; the oldest is completed
                                       when a fourth is launched); lms_sync and reads complete
                                       them in order.  Stream order keeps window state exact. */
#define LMS_FLAG_NVLS         0x8u  /* num_gpus > 1, LR2S / CM1*: merge the dense partial tables
                                       through NVLink-switch multicast (NVLS, multimem.red) when
                                       every device can join a multicast object; otherwise (or
                                       without the flag) the owner-push exchange (lms_nvls_active) */
#define LMS_FLAG_DENSE_VEHICLES 0x4u /* LR1: vehicle ids index the per-pane counts directly
                                       (VID < max_keys) instead of the key dictionary.  A record
                                       with VID >= max_keys is rejected: dropped, counted in
                                       overflow_records, and its batch completes with
                                       LMS_EINVAL.  Always on for multi-GPU LR1.              */

/* One aggregate result row (LR2S, CM1S, CM1T, CM2S) of window instance
 * [win_start_s, win_end_s) (readings R5/R6 in DESIGN.md).                    */
typedef struct {
  int64_t  win_start_s;
  int64_t  win_end_s;
  uint64_t key;        /* LR2: (xway*2+dir)*100+seg; CM1: category; CM2: jobId  */
  uint64_t count;      /* COUNT(*) of the group                                */
  uint64_t sum_fixed;  /* exact integer sum: LR2 speed; CM cpu * 1e6            */
  double   sum;        /* fp64 SUM (LR2 speed, CM cpu)                          */
  double   avg;        /* fp64 AVG = sum / count                                */
  uint32_t key_xway, key_dir, key_seg;  /* LR2 key decomposed                  */
  uint32_t rank;       /* CM1: position under ORDER BY SUM(cpu), ties by category */
} lms_agg_row;         /* 72 bytes */

/* One LR1 output row: an L record of the instance's newest slide with the
 * bag multiplicity m of its vehicle in the instance (reading R8).            */
typedef struct {
  int64_t  win_start_s;
  uint64_t vehicle;
  uint32_t ts;
  uint32_t multiplicity;
  uint16_t speed, xway, segment;
  uint8_t  lane, dir;
} lms_lr1_row;         /* 32 bytes */

/* Per-micro-batch record (SPEC S:64-69 fields plus device-side counters).   */
typedef struct {
  uint64_t index;            /* batch i                                          */
  uint64_t num_datasets;     /* NumDS_i                                          */
  uint64_t num_records;      /* records framed                                   */
  uint64_t batch_bytes;      /* sum_j Part_(i,j)                                 */
  double   admit_time_s;     /* caller clock at admission                        */
  double   max_buff_s;       /* max_j Buff_(i,j) = admit - ingest                */
  double   proc_s;           /* Proc_i: device time, admit -> results on host    */
  double   device_s;         /* kernels only (CUDA events)                       */
  double   h2d_s;            /* host->device copies of this batch's datasets     */
  double   d2h_s;            /* result rows device->host                         */
  double   max_lat_s;        /* Eq. 5: max_buff_s + proc_s                       */
  double   est_max_lat_s;    /* Eq. 6 at admission (NaN if bootstrap/forced)     */
  double   avg_thput_Bps;    /* Eq. 4 after this batch                           */
  double   inf_pt_bytes;     /* InfPT_i used by Alg. 2                           */
  uint32_t n_cpu_ops, n_gpu_ops;  /* Alg. 2 labels (report-only)                 */
  uint32_t plan_mask;        /* bit o = 1: op o labelled GPU                     */
  uint32_t admit_reason;     /* LMS_ADMIT_*                                      */
  double   plan_overhead_s;  /* host time in Alg. 2                              */
  double   admit_overhead_s; /* host time in Alg. 1                              */
  uint64_t windows_closed;
  uint64_t rows_emitted;
  uint64_t late_records;
  uint64_t bad_records;
  uint64_t overflow_records;
  int64_t  watermark;        /* max ts seen (-1: none)                           */
  double   opt_overhead_s;   /* LMS_FLAG_ONLINE_INFPT: duration of the Eq. 10 refit that
                                produced this batch's InfPT (run on the handle's worker
                                thread after the previous batch completed)      */
  double   opt_block_s;      /* time this batch's launch waited for that refit (Table V
                                "optimization blocking"); 0 when it had finished   */
} lms_batch_record;

enum { LMS_ADMIT_FORCED = 0, LMS_ADMIT_BOOTSTRAP = 1, LMS_ADMIT_TARGET = 2,
       LMS_ADMIT_TUMBLING_BOOTSTRAP = 3, LMS_ADMIT_CAP = 4, LMS_ADMIT_TRIGGER = 5,
       LMS_ADMIT_FLUSH = 6 };

/* Query DAG for Alg. 2 (CSR predecessor lists; the unique sink is the root). */
typedef struct {
  uint32_t n;
  const uint8_t* op_kind;      /* [n] lms_op_kind                                 */
  const int32_t* pred_off;     /* [n+1]                                            */
  const int32_t* preds;        /* [pred_off[n]]                                    */
} lms_dag;

/* ------------------------------------------------------------------ lifecycle */
uint32_t    lms_abi_version(void);
const char* lms_last_error(void);
/* Fill cfg with the defaults of query kind (Table IV window, Table III / P:733
 * constants).  Returns LMS_EINVAL for an unknown kind.                        */
lms_status  lms_config_init(lms_config* cfg, int32_t kind);
/* Validate cfg, allocate device state on cfg->device.  *out owned by the
 * library until lms_query_destroy.  Needs a CUDA device (LMS_ECUDA if none). */
lms_status  lms_query_create(const lms_config* cfg, lms_query** out);
lms_status  lms_query_destroy(lms_query* q);          /* NULL is a no-op        */

/* ------------------------------------------------------------------ ingest */
/* Push one dataset (whole records: LR nbytes % 70 == 0; CM ends with '\n').
 * The bytes are copied to device memory before return (the caller's buffer is
 * free on return); pinned caller memory takes the direct DMA path.
 * ingest_time_s must be non-decreasing.  nbytes > 0.  The datasets buffered for
 * one micro-batch (host-pushed and borrowed together) may total at most 2^37 B:
 * beyond it LMS_EOVERFLOW (admit what is buffered first); host-pushed bytes are
 * also bounded by cfg.max_batch_bytes (LMS_EOVERFLOW).                        */
lms_status  lms_push(lms_query* q, const void* bytes, uint64_t nbytes, double ingest_time_s,
                     uint64_t* dataset_id_out);
/* Asynchronous push of a dataset in PAGE-LOCKED host memory (cudaHostAlloc'd or
 * cudaHostRegister'ed; else LMS_EINVAL): the H2D copy into the library's staging
 * buffer is enqueued on the handle's copy stream and the call returns at once, so
 * the copy of the next micro-batch overlaps the kernels of the running one (the
 * batch's kernels wait for it on the device).  The host buffer is BORROWED until
 * the batch containing the dataset completes (lms_sync / a later lms_poll); its
 * device-timed H2D is reported in the batch record's h2d_s.  Same checks and caps
 * as lms_push.                                                                */
lms_status  lms_push_pinned(lms_query* q, const void* bytes, uint64_t nbytes, double ingest_time_s,
                            uint64_t* dataset_id_out);
/* Push a dataset already in device memory of the query's device (16-byte
 * aligned).  The buffer is BORROWED until the batch containing it completes
 * (lms_sync / a later lms_poll returns).  Same 2^37 B per-batch cap as lms_push. */
lms_status  lms_push_device(lms_query* q, const void* dptr, uint64_t nbytes, double ingest_time_s,
                            uint64_t* dataset_id_out);

/* ------------------------------------------------------------------ batches */
/* Alg. 1 poll at caller time now_s (call every 10 ms).  Completes a
 * finished in-flight batch first.  *admitted = 1 if a batch was admitted and
 * launched (asynchronously); *batch_index its index.                          */
lms_status  lms_poll(lms_query* q, double now_s, int32_t* admitted, uint64_t* batch_index);
/* Admit everything buffered now (MANUAL / TRIGGER, or any mode).  LMS_ESTATE
 * if a batch is still in flight (call lms_sync first).  *batch_index = the
 * new batch, or UINT64_MAX if nothing was buffered.                           */
lms_status  lms_force_batch(lms_query* q, double now_s, uint64_t* batch_index);
/* Admit the rest (if any) and close every remaining window (end of stream).  */
lms_status  lms_flush(lms_query* q, double now_s);
/* Wait for the in-flight batch (no-op if none); move its rows to the host
 * queue and fill its batch record.  Returns LMS_EFORMAT if it contained
 * malformed records, LMS_EOVERFLOW if a capacity was exceeded, LMS_EINVAL if a
 * dense-vehicle LR1 batch held a VID >= max_keys (rows of the valid records
 * are still delivered in every case).                                        */
lms_status  lms_sync(lms_query* q);

/* ------------------------------------------------------------------ results */
lms_status  lms_read_agg(lms_query* q, lms_agg_row* rows, uint64_t cap, uint64_t* n,
                         uint64_t* remaining);
lms_status  lms_read_lr1(lms_query* q, lms_lr1_row* rows, uint64_t cap, uint64_t* n,
                         uint64_t* remaining);
lms_status  lms_num_batches(lms_query* q, uint64_t* n);
lms_status  lms_get_batch_record(lms_query* q, uint64_t batch_index, lms_batch_record* out);

/* ------------------------------------------------------------------ multi-GPU (world > 1)
 * One handle per GPU / rank; the caller owns the collectives (NCCL via torch.distributed in
 * paper_2111_04289_b200/dist.py).  Per micro-batch:
 *   lms_force_batch / lms_poll   admit + launch the aggregate pass only (rank-local rows)
 *   all-reduce MAX of *wm, MIN of *ts_min on `stream` (lms_watermark_ptrs): one global
 *                                watermark (reading R7) on every rank
 *   lms_close_range (optional)   the instances this batch closes, identical on every rank
 *                                (syncs the stream); when none closes the caller may skip
 *                                the exchange: lms_run_close + lms_sync finish the batch
 *   lms_run_close                close windows as PARTIAL rows (count, exact sum, no HAVING /
 *                                rank) bucketed by owner rank = fmix64(key) % world
 *   lms_sync                     wait; partial rows stay on the device
 *   lms_partials                 device pointer of the bucketed rows + per-owner counts
 *   all-to-all of the rows (lms_agg_row bytes)
 *   lms_merge                    owner merge of the received rows -> final rows (AVG,
 *                                HAVING, ORDER BY rank) -> host row FIFO (lms_read_agg)   */
/* Device pointers of the live watermark (max kept ts + 1, 0 = none; u64) and of the batch's
 * minimum kept ts (u64, 0xFFFFFFFF = none), and the handle's cudaStream_t.               */
lms_status  lms_watermark_ptrs(lms_query* q, void** wm_dptr, void** tsmin_dptr, void** stream);
/* [k_first, k_last]: window instances [k*S, k*S + R) the pending close emits (empty when
 * k_last < k_first), from the all-reduced watermark (reading R7); call after the watermark
 * all-reduce, before lms_run_close.  ESTATE: single-GPU handle or no pending close.      */
lms_status  lms_close_range(lms_query* q, int64_t* k_first, int64_t* k_last);
lms_status  lms_run_close(lms_query* q);
lms_status  lms_partials(lms_query* q, const void** rows_dptr, uint64_t* counts /*[world]*/);
lms_status  lms_merge(lms_query* q, const void* rows_dptr, uint64_t n_rows);

/* Fused exchange (PAPER.md "Shuffling" Table III): replaces the
 * all-to-all + lms_merge steps for LR2S / CM1* / CM2S.  Every rank maps every other rank's
 * owner-side merge accumulators, key dictionary and state into its address space (CUDA IPC:
 * peer memory over NVLink/NVSwitch on a multi-GPU node; the same device works too), and a
 * kernel adds the rank's partial (exact sum, count) of each (instance, key) straight into the
 * owner's accumulators with remote RED.64 (CM2 keys: remote CAS in the owner's dictionary).
 * Setup once: lms_p2p_export -> exchange the handles (e.g. all_gather) -> lms_p2p_import of
 * every rank's handle (including the own one); in one process, lms_p2p_import_local(q, peer).
 * Per batch that closes windows, after lms_run_close + lms_sync, for each pass of at most
 * lms_merge_window instances [k_lo, k_lo + nwin) of [close k_first, k_last]:
 *   lms_p2p_push(k_lo, nwin) on every rank (returns when the pushes are complete)
 *   barrier across ranks
 *   lms_p2p_finalize(k_lo, nwin) on every rank: AVG / HAVING / ORDER BY rank of the keys it
 *                     owns -> host row FIFO (lms_read_agg)
 *   barrier across ranks (before the next pass or batch pushes again)
 * The handle is plain bytes (safe to send between processes).  EINVAL: null arguments, a peer
 * of another query shape; ESTATE: not a multi-GPU aggregate handle, peers not imported, batch
 * not complete; ECUDA: IPC failure (e.g. no peer access between the devices).            */
typedef struct {
  uint32_t rank, world, K, kind;
  uint64_t dict_cap_mask;
  uint32_t dict_max_keys, present;   /* present: bit i = ipc[i] is valid                  */
  uint8_t  ipc[6][64];               /* cudaIpcMemHandle_t of: merge sums, merge counts,
                                        dictionary {key, index} entries, dictionary free-
                                        index stack, keys by index, state (CM2 only: the
                                        dictionary slots ipc[2..4])                        */
} lms_p2p_handle;
lms_status  lms_p2p_export(lms_query* q, lms_p2p_handle* out);
lms_status  lms_p2p_import(lms_query* q, const lms_p2p_handle* peer);
lms_status  lms_p2p_import_local(lms_query* q, lms_query* peer);
lms_status  lms_merge_window(lms_query* q, uint32_t* wmerge);
/* Instances [k_first, k_last] the last completed batch closed (k_last < k_first: none).     */
lms_status  lms_last_close_range(lms_query* q, int64_t* k_first, int64_t* k_last);
lms_status  lms_p2p_push(lms_query* q, int64_t k_lo, uint32_t nwin);
lms_status  lms_p2p_finalize(lms_query* q, int64_t k_lo, uint32_t nwin);
/* Fully device-side variant (no host round trip inside the batch): after lms_run_close, and
 * without lms_sync, lms_p2p_exchange_async enqueues on the handle's stream: push of the
 * partials of the close's instances (at most lms_merge_window of them) into the owners'
 * accumulators -> device barrier (every rank bumps every rank's arrival counter through peer
 * memory; the owner's finalize waits for world arrivals) -> owner finalize -> completion
 * signal to every rank (the next exchange's pushes wait for it).  A batch that closes nothing
 * does nothing (identical on every rank).  lms_p2p_collect then completes the batch (the one
 * host synchronisation) and moves the owner's final rows to the host FIFO; instances beyond
 * the merge window (a long flush) are left to lms_p2p_push / lms_p2p_finalize passes
 * (lms_last_close_range).  Waits are bounded (20 s): a missing peer gives LMS_ECUDA, never a
 * hang.  ESTATE: not after lms_run_close, or a previous exchange not collected.            */
lms_status  lms_p2p_exchange_async(lms_query* q);
lms_status  lms_p2p_collect(lms_query* q);
/* enable != 0 (after lms_p2p_import of every rank; agg kinds): the watermark / first-ts
 * all-reduce (reading R7) also moves to the device — a one-thread kernel after the aggregate
 * pass folds this rank's values into every rank's slot through peer memory and waits for all
 * ranks (bounded) — so lms_force_batch enqueues aggregate, watermark exchange and close
 * without the caller's collective or lms_run_close; with lms_p2p_exchange_async +
 * lms_p2p_collect a whole multi-GPU micro-batch runs with one host synchronisation and no
 * per-batch NCCL call.  ESTATE: batch in flight, peers not imported.                       */
lms_status  lms_p2p_device_watermark(lms_query* q, int32_t enable);
/* *active = 1 iff this single-handle multi-device query (num_gpus > 1, LR2S / CM1S / CM1T)
 * merges its dense partial tables through NVLS (PAPER.md P:751, P:962 —
 * the shuffle): the merge accumulators of all devices are the replicas of one NVLink-switch
 * multicast object, the close's partial rows are reduced into every replica with
 * multimem.red.add.u64, and each key's owner finalizes it from its local replica and zeroes it
 * in all replicas with multimem.st — no owner push, no all-to-all.  0: the owner-push exchange
 * (no LMS_FLAG_NVLS, a device that cannot join a multicast object, CM2S / LR1, one GPU).   */
lms_status  lms_nvls_active(lms_query* q, int32_t* active);
/* Dense exchange (the small key sets — LR2 2000 keys, CM1 10 categories — are
 * reduced as dense arrays, PAPER.md P:751 / P:962 "shuffle"): after lms_run_close + lms_sync
 * of a batch that closed instances, for each merge window [k_lo, k_lo + nwin) (nwin <= the
 * merge window, lms_merge_window; instances from lms_last_close_range):
 *   lms_dense_partials  adds THIS rank's partial rows of those instances (all keys) into its
 *                       merge accumulators and returns them: *sum_dptr / *cnt_dptr = u64
 *                       [nwin][K] device arrays (row-major, K = the query's key space) of
 *                       *n_elems = nwin * K elements, owned by the library;
 *   (the caller SUM-all-reduces both arrays over the ranks, on the library's stream)
 *   lms_dense_finalize  rank 0 finalizes every key (AVG, HAVING avg < 40, CM1 rank) into its
 *                       row FIFO (rows_emitted of the batch record) and clears its arrays; the
 *                       other ranks clear theirs and emit nothing.
 * ESTATE: not a multi-GPU LR2S / CM1S / CM1T handle, or batch not complete; EINVAL: nwin.   */
lms_status  lms_dense_partials(lms_query* q, int64_t k_lo, uint32_t nwin, void** sum_dptr, void** cnt_dptr,
                               uint64_t* n_elems);
lms_status  lms_dense_finalize(lms_query* q, int64_t k_lo, uint32_t nwin);

/* Multi-GPU LR1 (LR1S / LR1T with world > 1; Table IV, reading R8).  Vehicles
 * index the per-pane counts directly (VID < max_keys; a larger VID is rejected: LMS_EINVAL), every
 * rank keeps and probes its own rows, and the multiplicity m of a probed row counts the
 * vehicle in the whole window over ALL ranks.  Per micro-batch, after the watermark
 * all-reduce and before lms_run_close:
 *   lms_close_range       instances [k_first, k_last] this batch closes (above)
 *   for each k:  lms_lr1_window_counts(k) -> device uint32[n_counts] of this rank's counts
 *                of instance k per vehicle; the caller all-reduces it (SUM) on `stream`;
 *                lms_lr1_probe(k) emits the rows of instance k (newest slide) with the
 *                all-reduced m
 *   lms_run_close, lms_sync: state update / eviction; rows are final -> lms_read_lr1.
 * The counts buffer is library-owned and reused by the next call.  EINVAL: null arguments;
 * ESTATE: not a multi-GPU LR1 handle, or no aggregate pass awaiting its close.          */
lms_status  lms_lr1_window_counts(lms_query* q, int64_t k, void** counts_dptr, uint64_t* n_counts);
lms_status  lms_lr1_probe(lms_query* q, int64_t k);

/* Record-boundary row partition of one dataset for `parts` GPUs (the paper's
 * partitioning of a micro-batch): offsets[0..parts] (caller-owned, parts + 1 entries),
 * offsets[0] = 0, offsets[parts] = nbytes, non-decreasing, every range whole records.  LR
 * (kind LR*): cut i = the 70 B multiple at or below i*nbytes/parts.  CM: cut i = the first
 * byte after a '\n' at or after i*nbytes/parts (a part may be empty when records are longer
 * than nbytes/parts).  `bytes` may be host or device memory (device: only the bytes around
 * each cut are read).  EINVAL: null / empty, LR size not a multiple of 70, CM not ending in
 * '\n'.                                                                                   */
lms_status  lms_split(int32_t kind, const void* bytes, uint64_t nbytes, uint32_t parts, uint64_t* offsets);

/* ------------------------------------------------------------------ timing hooks */
/* Device time of the last completed batch's kernels, and of its dominant
 * kernel (aggregate pass) alone, in seconds (CUDA events on the query stream). */
lms_status  lms_last_kernel_times(lms_query* q, double* batch_s, double* agg_s, double* close_s);
/* Number of kernels the library launched so far (all batches).              */
lms_status  lms_kernel_launches(lms_query* q, uint64_t* n);

/* ------------------------------------------------------------------ pure cost models */
/* Eq. 6: max_j buff_s[j] + (sum_j bytes[j]) / avg_thput.  n >= 1,
 * avg_thput > 0 else LMS_EINVAL.                                              */
lms_status  lms_est_max_lat(const double* buff_s, const uint64_t* bytes, uint64_t n,
                            double avg_thput, double* out);
/* Eq. 7 / 8 / 9.  Non-positive inputs -> LMS_EINVAL.   */
lms_status  lms_cpu_cost(double base, double part, double infpt, double* out);
lms_status  lms_gpu_cost(double base, double part, double infpt, double* out);
lms_status  lms_trans_cost(double btc, double part, double infpt, double* out);
/* Table III base cost of an operation kind.                      */
lms_status  lms_base_cost(int32_t op_kind, double* out);
/* Alg. 2: dev_out[o] = LMS_DEV_CPU / LMS_DEV_GPU.  LMS_EPLAN on a
 * cycle or multiple roots.                                                    */
lms_status  lms_map_device(const lms_dag* dag, double part_bytes, double infpt, double btc,
                           uint8_t* dev_out);
/* Canonical DAG of a query kind.  Arrays are library-owned.      */
lms_status  lms_query_dag(int32_t kind, lms_dag* out);
/* Alg. 1 decision for one poll (pure; P:625-689 + readings R11/R15/R22):
 *   ingest_s/bytes: tmp = buffered U new, already in creation order (n >= 0);
 *   avg_thput <= 0 means "no completed batch yet" (bootstrap, admit);
 *   maxlat_hist: MaxLat of completed batches (tumbling target = their mean).
 *   mode: LMS_MODE_LMSTREAM or LMS_MODE_DEADLINE.
 * *admit = 0/1; *est = EstMaxLat (NaN if not computed); *reason = LMS_ADMIT_*
 * or -1 for "buffer" / -2 for "poll" (nothing to judge).                     */
lms_status  lms_admit_decision(int32_t mode, double slide_s, double deadline_s, double now_s,
                               const double* ingest_s, const uint64_t* bytes, uint64_t n,
                               double avg_thput, const double* maxlat_hist, uint64_t n_hist,
                               int32_t* admit, double* est, int32_t* reason);
/* Eq. 10 OLS fit over rows (thput_Bps, lat_s, infpt_bytes); LMS_EHISTORY if
 * < 3 rows or singular.  predict clamps to [1 KiB, 16 MiB].                  */
lms_status  lms_infpt_fit(const double* thput_Bps, const double* lat_s, const double* infpt,
                          uint64_t n, double* b0, double* b1, double* b2);
lms_status  lms_infpt_predict(double b0, double b1, double b2, double thput_Bps, double lat_s,
                              double* out);
/* Nearest-rank percentile of n values.                               */
lms_status  lms_percentile(const double* v, uint64_t n, double p, double* out);

#ifdef __cplusplus
}
#endif
#endif /* LMSTREAM_H */
