"""Multi-GPU execution: row-partitioned micro-batches + partial-aggregate exchange.

PAPER.md: the micro-batch is split into partitions processed in parallel and the
partial aggregates are shuffled before the final aggregation ("Shuffling", Table III P:751;
"shuffle aggregate" P:962).  Here one process drives one GPU (torchrun; NCCL via
torch.distributed — PyTorch is the process-group plumbing only).  Every rank owns one
lms_query (lms_config.rank/world) and processes its own rows of each micro-batch; per batch:

  1. lms_force_batch          aggregate pass over the rank's rows (CUDA kernel)
  2. all-reduce MAX / MIN      global watermark and first-batch ts_min (reading R7) — NCCL on
                               the handle's stream, no host round trip
  3. lms_run_close             partial rows of the closing instances, bucketed by owner rank
                               (kernels)
  4. lms_sync                  wait
  5. all-to-all                partial rows to their owners (NCCL, bytes of lms_agg_row)
  6. lms_merge                 owner-side merge + AVG / HAVING / ORDER BY rank (kernels)

LR1 (self-join, no owner exchange): after step 2, for every instance the batch closes the
ranks' vehicle-indexed window counts are all-reduced (SUM, 4 B per vehicle) and each rank
probes its own newest-slide rows against the global counts (lms_lr1_* calls).

`Exchange` implementation: TorchDistExchange (one handle per process, any torch.distributed
backend: NCCL on GPUs, gloo for the CPU protocol tests).  The tests' LocalExchange
(tests/local_exchange.py: several handles on one GPU in one process, "virtual shards") drives
the same protocol without a process group.  run_batch(p2p=True) uses the fused exchange instead: each rank
adds its partials straight into the owners' accumulators through peer-mapped memory (CUDA IPC
over NVLink; lms_p2p_*), then barrier + owner finalize — no all-to-all, no merge copy.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from ._lib import check

ROW_BYTES = C.sizeof(L.lms_agg_row)


class _CudaPtr:
    """Raw device pointer exposed through __cuda_array_interface__ (for torch.as_tensor)."""

    def __init__(self, ptr: int, nbytes: int, typestr: str = "|u1", itemsize: int = 1):
        self.__cuda_array_interface__ = {"shape": (nbytes // itemsize,), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def device_view(ptr: int, nbytes: int, dtype="u1"):
    import torch
    typestr, size = {"u1": ("|u1", 1), "i4": ("<i4", 4), "i8": ("<i8", 8)}[dtype]
    if nbytes == 0:
        return torch.empty(0, dtype={"u1": torch.uint8, "i4": torch.int32, "i8": torch.int64}[dtype], device="cuda")
    return torch.as_tensor(_CudaPtr(ptr, nbytes, typestr, size), device="cuda")


# ----------------------------------------------------------------------------- host split

def split_points(family: str, data, world: int) -> list[tuple[int, int]]:
    """Row partition of one dataset at record boundaries: [(offset, nbytes)] per rank, computed
    by the library (lms_split).  data: bytes-like host memory, or (pointer, nbytes) of host or
    device memory."""
    if isinstance(data, tuple):
        ptr, n = data
        keep = None
    else:
        arr = np.frombuffer(data, dtype=np.uint8) if not isinstance(data, np.ndarray) else data
        arr = np.ascontiguousarray(arr)
        ptr, n, keep = arr.ctypes.data, arr.nbytes, arr
    offs = (C.c_uint64 * (world + 1))()
    kind = L.LMS_LR2S if family == "LR" else L.LMS_CM2S
    check(L.lms_split(kind, C.c_void_p(ptr), n, world, offs), "lms_split")
    del keep
    return [(offs[i], offs[i + 1] - offs[i]) for i in range(world)]


# ----------------------------------------------------------------------------- handles

class RankHandle:
    """One rank's lms_query plus typed views of its protocol buffers."""

    def __init__(self, query):
        self.q = query
        self.world = query.cfg.world
        wm, tsmin, stream = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(L.lms_watermark_ptrs(query.h, C.byref(wm), C.byref(tsmin), C.byref(stream)), "lms_watermark_ptrs")
        self.wm_ptr, self.tsmin_ptr, self.stream_ptr = wm.value, tsmin.value, stream.value or 0

    def watermark_tensors(self):
        return device_view(self.wm_ptr, 8, "i8"), device_view(self.tsmin_ptr, 8, "i8")

    def partials(self):
        """(uint8 device tensor of the bucketed partial rows, per-owner row counts)."""
        ptr = C.c_void_p()
        counts = (C.c_uint64 * self.world)()
        check(L.lms_partials(self.q.h, C.byref(ptr), counts), "lms_partials")
        cnt = [int(c) for c in counts]
        return device_view(ptr.value or 0, sum(cnt) * ROW_BYTES), cnt

    def windows_closed(self) -> int:
        """Window instances the last completed batch closed (identical on every rank)."""
        return self.q.record(self.q.num_batches() - 1)["windows_closed"]

    # ---- fused exchange (peer-mapped owner accumulators)
    def p2p_export(self) -> bytes:
        h = L.lms_p2p_handle()
        check(L.lms_p2p_export(self.q.h, C.byref(h)), "lms_p2p_export")
        return bytes(h)

    def p2p_import(self, blob: bytes):
        h = L.lms_p2p_handle.from_buffer_copy(blob)
        check(L.lms_p2p_import(self.q.h, C.byref(h)), "lms_p2p_import")

    def p2p_import_local(self, other: "RankHandle"):
        check(L.lms_p2p_import_local(self.q.h, other.q.h), "lms_p2p_import_local")

    def merge_window(self) -> int:
        w = C.c_uint32()
        check(L.lms_merge_window(self.q.h, C.byref(w)), "lms_merge_window")
        return w.value

    def last_close_range(self):
        k0, k1 = C.c_int64(), C.c_int64()
        check(L.lms_last_close_range(self.q.h, C.byref(k0), C.byref(k1)), "lms_last_close_range")
        return k0.value, k1.value

    def p2p_push(self, k_lo: int, nwin: int):
        check(L.lms_p2p_push(self.q.h, k_lo, nwin), "lms_p2p_push")

    def p2p_exchange_async(self):
        check(L.lms_p2p_exchange_async(self.q.h), "lms_p2p_exchange_async")

    def p2p_device_watermark(self, enable: bool = True):
        check(L.lms_p2p_device_watermark(self.q.h, int(enable)), "lms_p2p_device_watermark")

    def p2p_collect(self) -> int:
        return check(L.lms_p2p_collect(self.q.h), "lms_p2p_collect", (L.LMS_OK, L.LMS_EFORMAT, L.LMS_EOVERFLOW))

    def p2p_finalize(self, k_lo: int, nwin: int):
        return check(L.lms_p2p_finalize(self.q.h, k_lo, nwin), "lms_p2p_finalize", (L.LMS_OK, L.LMS_EOVERFLOW))

    def close_range(self):
        """Window instances [k0, k1] the pending close emits (k1 < k0: none)."""
        k0, k1 = C.c_int64(), C.c_int64()
        check(L.lms_close_range(self.q.h, C.byref(k0), C.byref(k1)), "lms_close_range")
        return k0.value, k1.value

    # ---- multi-GPU LR1
    def lr1_window_counts(self, k: int):
        """int32 device view of this rank's vehicle counts of instance k (all-reduce it: SUM)."""
        ptr, n = C.c_void_p(), C.c_uint64()
        check(L.lms_lr1_window_counts(self.q.h, k, C.byref(ptr), C.byref(n)), "lms_lr1_window_counts")
        return device_view(ptr.value, n.value * 4, "i4")

    def lr1_probe(self, k: int):
        check(L.lms_lr1_probe(self.q.h, k), "lms_lr1_probe")

    def run_close(self):
        check(L.lms_run_close(self.q.h), "lms_run_close")

    def sync(self) -> int:
        return self.q.sync(ok=(L.LMS_OK, L.LMS_EFORMAT, L.LMS_EOVERFLOW))

    # ---- dense exchange (LR2S / CM1*: small key sets reduced as dense arrays)
    def dense_partials(self, k_lo: int, nwin: int):
        """int64 device views of this rank's merge accumulators [nwin][K] (sums, counts) after
        its own partial rows of instances [k_lo, k_lo + nwin) were added (all-reduce: SUM)."""
        s, c, n = C.c_void_p(), C.c_void_p(), C.c_uint64()
        check(L.lms_dense_partials(self.q.h, k_lo, nwin, C.byref(s), C.byref(c), C.byref(n)), "lms_dense_partials")
        return device_view(s.value, n.value * 8, "i8"), device_view(c.value, n.value * 8, "i8")

    def dense_finalize(self, k_lo: int, nwin: int):
        return check(L.lms_dense_finalize(self.q.h, k_lo, nwin), "lms_dense_finalize", (L.LMS_OK, L.LMS_EOVERFLOW))

    def merge(self, rows_u8):
        n = rows_u8.numel() // ROW_BYTES
        ptr = rows_u8.data_ptr() if n else None
        return check(L.lms_merge(self.q.h, C.c_void_p(ptr), n), "lms_merge", (L.LMS_OK, L.LMS_EOVERFLOW))


# ----------------------------------------------------------------------------- exchanges

class TorchDistExchange:
    """torch.distributed collectives (one handle per process)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # gloo (CPU protocol tests, or ranks sharing one GPU in tests): stage device tensors
        # through host memory; NCCL runs on the library's stream directly
        self.host_staged = dist.get_backend(group) == "gloo"

    def _all_reduce(self, t, op):
        if self.host_staged and t.is_cuda:
            import torch
            torch.cuda.synchronize()
            c = t.cpu()
            self.dist.all_reduce(c, op=op, group=self.group)
            t.copy_(c)
            torch.cuda.synchronize()
        else:
            self.dist.all_reduce(t, op=op, group=self.group)

    def _a2a(self, out, inp, out_splits=None, in_splits=None):
        if self.host_staged and inp.is_cuda:
            import torch
            torch.cuda.synchronize()
            co = torch.empty(out.shape, dtype=out.dtype)
            self.dist.all_to_all_single(co, inp.cpu(), output_split_sizes=out_splits,
                                        input_split_sizes=in_splits, group=self.group)
            out.copy_(co)
            torch.cuda.synchronize()
        else:
            self.dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits,
                                        group=self.group)

    def _on(self, h):
        import torch
        if h is None or not getattr(h, "stream_ptr", 0):
            return _Null()
        return torch.cuda.stream(torch.cuda.ExternalStream(h.stream_ptr))

    def allreduce_watermarks(self, handles):
        """In place on the library's state: MAX all-reduce of the watermark, MIN of the batch's
        first ts (reading R7) — collectives only, no compute outside the library."""
        (h,) = handles
        wm, tsmin = h.watermark_tensors()
        with self._on(h):
            self._all_reduce(wm, self.dist.ReduceOp.MAX)
            self._all_reduce(tsmin, self.dist.ReduceOp.MIN)

    def setup_p2p(self, handles, device_watermark: bool = False):
        """Fused exchange: every rank maps every rank's owner state (CUDA IPC handles sent with
        all_gather_object)."""
        (h,) = handles
        blobs = [None] * self.world
        self.dist.all_gather_object(blobs, h.p2p_export(), group=self.group)
        for b in blobs:
            h.p2p_import(b)
        if device_watermark:
            h.p2p_device_watermark(True)

    def barrier(self, handles):
        self.dist.barrier(group=self.group)

    def allreduce_sum(self, handles, tensors):
        """In-place SUM all-reduce of tensors[0] (LR1 window counts) on the handle's stream."""
        (h,), (t,) = handles, tensors
        with self._on(h):
            self._all_reduce(t, self.dist.ReduceOp.SUM)

    def allreduce_dense(self, handles, arrays):
        """In-place SUM all-reduce of arrays[0] = (sums, counts) on the handle's stream."""
        (h,), ((sums, cnts),) = handles, arrays
        with self._on(h):
            self._all_reduce(sums, self.dist.ReduceOp.SUM)
            self._all_reduce(cnts, self.dist.ReduceOp.SUM)

    def all_to_all(self, handles, sends):
        """sends[0] = (uint8 rows tensor grouped by owner, per-owner counts) -> received rows."""
        import torch
        (h,), ((rows, counts),) = handles, sends
        dev = rows.device
        send_c = torch.tensor(counts, dtype=torch.int64, device=dev)
        recv_c = torch.empty_like(send_c)
        with self._on(h):
            self._a2a(recv_c, send_c)
            rc = [int(x) for x in recv_c.tolist()]
            recv = torch.empty(sum(rc) * ROW_BYTES, dtype=torch.uint8, device=dev)
            self._a2a(recv, rows, [c * ROW_BYTES for c in rc], [c * ROW_BYTES for c in counts])
        return [recv]


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# ----------------------------------------------------------------------------- protocol

def run_batch(handles, exchange, now: float, flush: bool = False, p2p=False) -> list[int]:
    """One micro-batch on every local handle (steps 1-6 above; LR1: close_lr1's steps).
    p2p="dense" (LR2S / CM1*): the partial sums are reduced as dense [instances][K] arrays with
    one SUM all-reduce per merge window (small key sets) and rank 0 finalizes;
    p2p=True: fused exchange (exchange.setup_p2p done once) instead of all-to-all + lms_merge,
    host-driven passes; p2p="async": the same exchange fully enqueued behind the close with a
    device-side barrier (one host synchronisation per batch); p2p="device": in addition the
    watermark exchange runs on the device (handles set up with p2p_device_watermark), so no
    collective is issued per batch.  Returns the sync statuses."""
    for h in handles:
        st = L.lms_flush(h.q.h, now) if flush else L.lms_force_batch(h.q.h, now, None)
        check(st, "lms_flush" if flush else "lms_force_batch", (L.LMS_OK, L.LMS_EFORMAT))
    if p2p == "device":
        # aggregate, watermark exchange and close are already enqueued (device-side exchange)
        return _exchange_async(handles, exchange)
    exchange.allreduce_watermarks(handles)
    if handles[0].q.kind in (L.LMS_LR1S, L.LMS_LR1T):
        return close_lr1(handles, exchange)
    for h in handles:
        h.run_close()
    if p2p == "async":
        return _exchange_async(handles, exchange)
    sts = [h.sync() for h in handles]
    if handles[0].windows_closed() == 0:   # same on every rank: nothing to exchange (most batches)
        return sts
    if p2p == "dense":
        exchange_dense(handles, exchange)
        return sts
    if p2p:
        exchange_p2p(handles, exchange)
        return sts
    recvs = exchange.all_to_all(handles, [h.partials() for h in handles])
    for h, rows in zip(handles, recvs):
        h.merge(rows)
    return sts


def exchange_p2p(handles, exchange, k_from=None):
    """Fused exchange of a synced batch that closed windows: per merge-window pass, every rank
    pushes its partials into the owners' accumulators (peer memory), barrier, every owner
    finalizes its keys (rows -> host), barrier."""
    k0, k1 = handles[0].last_close_range()
    if k_from is not None:
        k0 = k_from
    wmerge = handles[0].merge_window()
    for k in range(k0, k1 + 1, wmerge):
        nwin = min(wmerge, k1 - k + 1)
        for h in handles:
            h.p2p_push(k, nwin)
        exchange.barrier(handles)
        for h in handles:
            h.p2p_finalize(k, nwin)
        exchange.barrier(handles)


def exchange_dense(handles, exchange):
    """Dense exchange of the last close's instances, one merge window at a time."""
    k0, k1 = handles[0].last_close_range()
    wmerge = handles[0].merge_window()
    k = k0
    while k <= k1:
        nwin = min(wmerge, k1 - k + 1)
        arrays = [h.dense_partials(k, nwin) for h in handles]
        exchange.allreduce_dense(handles, arrays)
        for h in handles:
            h.dense_finalize(k, nwin)
        k += nwin


def _exchange_async(handles, exchange):
    """Fused exchange fully enqueued behind the close: push -> device barrier -> owner
    finalize -> signal; one host synchronisation (collect) per rank."""
    for h in handles:
        h.p2p_exchange_async()
    sts = [h.p2p_collect() for h in handles]
    k0, k1 = handles[0].last_close_range()
    w = handles[0].merge_window()
    if k1 - k0 + 1 > w:                      # a long flush: the rest in host-driven passes
        exchange_p2p(handles, exchange, k_from=k0 + w)
    return sts


def _close_range(handles):
    k0, k1 = handles[0].close_range()
    for h in handles[1:]:
        assert h.close_range() == (k0, k1), "ranks disagree on the closing instances"
    return k0, k1


def close_lr1(handles, exchange) -> list[int]:
    """LR1 (window self-join, reading R8) on row-partitioned batches: for every instance the
    batch closes, each rank's vehicle counts of the window are all-reduced (SUM) and every rank
    probes its own newest-slide rows against them; the union of the ranks' rows is the
    single-GPU result.  No rows move between ranks."""
    k0, k1 = _close_range(handles)
    for k in range(k0, k1 + 1):
        exchange.allreduce_sum(handles, [h.lr1_window_counts(k) for h in handles])
        for h in handles:
            h.lr1_probe(k)
    for h in handles:
        h.run_close()
    return [h.sync() for h in handles]


# ----------------------------------------------------------------------------- admission

class DistAdmission:
    """Alg. 1 / CG(dN) for micro-batches partitioned across ranks.

    Every dataset arrives once and is split at record boundaries (lms_split): each rank
    registers its own partition with push(ingest_s, local_bytes), in the same order on every
    rank.  poll(now) sums the partitions' bytes over the ranks (one SUM all-reduce), rank 0
    judges the GLOBAL datasets with the library's Alg. 1 (lms_admit_decision: Eq. 6 EstMaxLat
    against SlideTime / the deadline / the mean past MaxLat) and broadcasts its decision, so
    every rank admits the same datasets at the same poll and then forces its partition
    (lms_force_batch).  complete(proc_local): a partitioned batch completes when its slowest
    partition does, so Proc is the MAX over ranks; rank 0's Eq. 4 (AvgThPut: global bytes over
    the running Proc sum) and Eq. 5 (MaxLat = max Buff + Proc) history drives the next poll.
    mode: L.LMS_MODE_LMSTREAM or L.LMS_MODE_DEADLINE (CG(dN): SlideTime := N, d0 tumbling)."""

    def __init__(self, mode: int, slide_s: float = 0.0, deadline_s: float = 0.0, group=None):
        import torch.distributed as dist
        if mode not in (L.LMS_MODE_LMSTREAM, L.LMS_MODE_DEADLINE):
            raise ValueError("DistAdmission runs Alg. 1 (LMS_MODE_LMSTREAM / LMS_MODE_DEADLINE)")
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
        self.mode, self.slide_s, self.deadline_s = mode, float(slide_s), float(deadline_s)
        self.buffered = []          # [(ingest_s, global bytes, local bytes)] judged, not admitted
        self.new = []               # [(ingest_s, local bytes)] since the last poll
        self.bytes_hist, self.proc_sum, self.maxlat_hist = 0, 0.0, []
        self.in_flight = None       # (admit time, [(ingest_s, global bytes, local bytes)])
        self.last_proc = float("nan")   # Proc of the last completed batch (max over ranks)

    @property
    def avg_thput(self) -> float:
        """Eq. 4 over the completed batches (0 before the first: bootstrap)."""
        return self.bytes_hist / self.proc_sum if self.proc_sum > 0 else 0.0

    def push(self, ingest_s: float, local_bytes: int):
        self.new.append((float(ingest_s), int(local_bytes)))

    def poll(self, now: float):
        """-> (admitted, n_datasets, est_max_lat, reason); the same on every rank."""
        import torch
        if self.in_flight is not None:
            return False, 0, float("nan"), -2
        new, self.new = self.new, []
        if new:                                   # global bytes of the new partitions
            t = torch.tensor([b for _, b in new], dtype=torch.int64, device=self.dev)
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
            glob = [int(x) for x in t.cpu().tolist()]
            # Alg. 1: tmp = buffered U new, new sorted by creation time (stable: arrival order)
            order = sorted(range(len(new)), key=lambda i: new[i][0])
            self.buffered += [(new[i][0], glob[i], new[i][1]) for i in order]
        dec = torch.zeros(3, dtype=torch.float64, device=self.dev)
        if self.rank == 0:
            admit, est, reason = self._decide(now)
            dec[0], dec[1], dec[2] = float(admit), est, float(reason)
        self.dist.broadcast(dec, src=0, group=self.group)
        d = dec.cpu().tolist()
        admitted, est, reason = bool(d[0]), d[1], int(d[2])
        if not admitted:
            return False, 0, est, reason
        batch, self.buffered = self.buffered, []
        self.in_flight = (float(now), batch)
        return True, len(batch), est, reason

    def _decide(self, now: float):
        n = len(self.buffered)
        ing = (C.c_double * max(1, n))(*[x for x, _, _ in self.buffered])
        byt = (C.c_uint64 * max(1, n))(*[b for _, b, _ in self.buffered])
        hist = (C.c_double * max(1, len(self.maxlat_hist)))(*self.maxlat_hist)
        admit, est, reason = C.c_int32(), C.c_double(), C.c_int32()
        check(L.lms_admit_decision(self.mode, self.slide_s, self.deadline_s, float(now), ing, byt, n,
                                   self.avg_thput, hist, len(self.maxlat_hist), C.byref(admit),
                                   C.byref(est), C.byref(reason)), "lms_admit_decision")
        return admit.value, est.value, reason.value

    @property
    def in_flight_local_bytes(self) -> int:
        """This rank's bytes of the admitted, not yet completed batch (its partition)."""
        return sum(b for _, _, b in self.in_flight[1]) if self.in_flight else 0

    def complete(self, proc_local: float) -> float:
        """The in-flight batch finished on this rank after proc_local seconds: Proc = max over
        ranks; returns the batch's MaxLat (Eq. 5)."""
        import torch
        now, batch = self.in_flight
        self.in_flight = None
        t = torch.tensor([float(proc_local)], dtype=torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        proc = float(t.cpu().item())
        self.last_proc = proc
        self.bytes_hist += sum(b for _, b, _ in batch)
        self.proc_sum += proc
        ml = max(now - x for x, _, _ in batch) + proc
        self.maxlat_hist.append(ml)
        return ml
