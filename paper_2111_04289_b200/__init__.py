"""paper_2111_04289_b200 — B200-native LMStream (arXiv 2111.04289) micro-batch hot path.

The product is ``liblmstream.so`` (C ABI: ``include/lmstream.h``; sources ``csrc/``).
``_lib`` is its ctypes binding (same function names); ``Query`` below is a thin
convenience wrapper (handle ownership, status checks, row arrays).  All compute
runs in the CUDA kernels of the library; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from ._lib import KIND, MODE, LmsError, check  # noqa: F401

AGG_DTYPE = np.dtype([("win_start_s", "<i8"), ("win_end_s", "<i8"), ("key", "<u8"), ("count", "<u8"),
                      ("sum_fixed", "<u8"), ("sum", "<f8"), ("avg", "<f8"), ("key_xway", "<u4"),
                      ("key_dir", "<u4"), ("key_seg", "<u4"), ("rank", "<u4")])
LR1_DTYPE = np.dtype([("win_start_s", "<i8"), ("vehicle", "<u8"), ("ts", "<u4"), ("multiplicity", "<u4"),
                      ("speed", "<u2"), ("xway", "<u2"), ("segment", "<u2"), ("lane", "u1"), ("dir", "u1")])
assert AGG_DTYPE.itemsize == C.sizeof(L.lms_agg_row) and LR1_DTYPE.itemsize == C.sizeof(L.lms_lr1_row)


def config(kind: str | int, **overrides) -> L.lms_config:
    """lms_config_init defaults + overrides (device_ids: a sequence of CUDA ordinals, kept alive
    on the returned struct as `_device_ids`; it implies num_gpus = len(device_ids))."""
    cfg = L.lms_config()
    k = KIND[kind.upper()] if isinstance(kind, str) else int(kind)
    check(L.lms_config_init(C.byref(cfg), k), "lms_config_init")
    for name, val in overrides.items():
        if name == "mode" and isinstance(val, str):
            val = MODE[val]
        if name == "device_ids" and val is not None:
            arr = (C.c_int32 * len(val))(*val)
            cfg._device_ids = arr
            cfg.num_gpus = len(val)
            val = C.cast(arr, C.POINTER(C.c_int32))
        setattr(cfg, name, val)
    return cfg


class Query:
    """Owns one lms_query handle."""

    def __init__(self, kind: str | int, **overrides):
        self.cfg = config(kind, **overrides)
        self.kind = self.cfg.kind
        h = C.c_void_p()
        check(L.lms_query_create(C.byref(self.cfg), C.byref(h)), "lms_query_create")
        self.h = h

    # -- lifecycle
    def close(self):
        if getattr(self, "h", None):
            L.lms_query_destroy(self.h)
            self.h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- ingest
    def push(self, data, ingest_time: float) -> int:
        """data: bytes / bytearray / numpy uint8 array / (host pointer, nbytes)."""
        did = C.c_uint64()
        if isinstance(data, tuple):
            ptr, n = data
        elif isinstance(data, np.ndarray):
            ptr, n = data.ctypes.data, data.nbytes
        else:
            buf = (C.c_char * len(data)).from_buffer_copy(data) if isinstance(data, bytes) else \
                (C.c_char * len(data)).from_buffer(data)
            ptr, n = C.addressof(buf), len(data)
        check(L.lms_push(self.h, C.c_void_p(ptr), n, ingest_time, C.byref(did)), "lms_push")
        return did.value

    def push_pinned(self, ptr: int, nbytes: int, ingest_time: float) -> int:
        """Asynchronous push of page-locked host memory (borrowed until its batch completes)."""
        did = C.c_uint64()
        check(L.lms_push_pinned(self.h, C.c_void_p(ptr), nbytes, ingest_time, C.byref(did)), "lms_push_pinned")
        return did.value

    def push_device(self, dptr: int, nbytes: int, ingest_time: float) -> int:
        did = C.c_uint64()
        check(L.lms_push_device(self.h, C.c_void_p(dptr), nbytes, ingest_time, C.byref(did)), "lms_push_device")
        return did.value

    # -- batches
    def poll(self, now: float, ok=(L.LMS_OK,)):
        adm, idx = C.c_int32(), C.c_uint64()
        st = check(L.lms_poll(self.h, now, C.byref(adm), C.byref(idx)), "lms_poll", ok)
        return (idx.value if adm.value else None), st

    def force(self, now: float):
        idx = C.c_uint64()
        check(L.lms_force_batch(self.h, now, C.byref(idx)), "lms_force_batch")
        return None if idx.value == 2 ** 64 - 1 else idx.value

    def sync(self, ok=(L.LMS_OK,)) -> int:
        return check(L.lms_sync(self.h), "lms_sync", ok)

    def flush(self, now: float, ok=(L.LMS_OK,)) -> int:
        return check(L.lms_flush(self.h, now), "lms_flush", ok)

    # -- results
    def _drain(self, fn, dtype, ctype, name, out=None):
        n, rem = C.c_uint64(), C.c_uint64()
        if out is not None:                     # caller-owned, reusable buffer: fill a prefix
            if out.dtype != dtype or not out.flags.c_contiguous:
                raise TypeError(f"out must be a C-contiguous {dtype} array")
            check(fn(self.h, out.ctypes.data_as(C.POINTER(ctype)), len(out), C.byref(n), C.byref(rem)), name)
            return out[:n.value]
        check(fn(self.h, None, 0, C.byref(n), C.byref(rem)), name)      # how many are queued
        arr = np.empty(rem.value, dtype)
        if rem.value:
            check(fn(self.h, arr.ctypes.data_as(C.POINTER(ctype)), rem.value, C.byref(n), C.byref(rem)), name)
        return arr[:n.value]

    def read_agg(self, out=None) -> np.ndarray:
        """Queued LR2 / CM1 / CM2 rows (FIFO).  out: optional reusable AGG_DTYPE buffer; then
        at most len(out) rows are read into it and a view of them is returned."""
        return self._drain(L.lms_read_agg, AGG_DTYPE, L.lms_agg_row, "lms_read_agg", out)

    def read_lr1(self, out=None) -> np.ndarray:
        return self._drain(L.lms_read_lr1, LR1_DTYPE, L.lms_lr1_row, "lms_read_lr1", out)

    def queued_rows(self) -> int:
        n, rem = C.c_uint64(), C.c_uint64()
        fn = L.lms_read_lr1 if self.kind in (L.LMS_LR1S, L.LMS_LR1T) else L.lms_read_agg
        check(fn(self.h, None, 0, C.byref(n), C.byref(rem)), "lms_read")
        return rem.value

    def num_batches(self) -> int:
        n = C.c_uint64()
        check(L.lms_num_batches(self.h, C.byref(n)), "lms_num_batches")
        return n.value

    def record(self, i: int) -> dict:
        r = L.lms_batch_record()
        check(L.lms_get_batch_record(self.h, i, C.byref(r)), "lms_get_batch_record")
        return {f: getattr(r, f) for f, _ in r._fields_}

    def records(self) -> list[dict]:
        return [self.record(i) for i in range(self.num_batches())]

    def kernel_times(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        check(L.lms_last_kernel_times(self.h, C.byref(a), C.byref(b), C.byref(c)), "lms_last_kernel_times")
        return a.value, b.value, c.value

    def kernel_launches(self) -> int:
        n = C.c_uint64()
        check(L.lms_kernel_launches(self.h, C.byref(n)), "lms_kernel_launches")
        return n.value


def percentile(values, p: float) -> float:
    """Nearest-rank percentile computed by the library (lms_percentile)."""
    v = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    out = C.c_double()
    check(L.lms_percentile(v.ctypes.data_as(C.POINTER(C.c_double)), len(v), float(p), C.byref(out)),
          "lms_percentile")
    return out.value
