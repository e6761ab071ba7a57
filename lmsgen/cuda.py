"""ctypes binding of lmsgen/liblmsgen.so (CUDA generator, byte-identical to lmsgen/__init__.py).

INPUT GENERATION ONLY — used by tests and bench.py to build large micro-batches in HBM.
"""
from __future__ import annotations

import ctypes as C
import os

from . import SEED, CMParams, LRParams, Traffic

_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "liblmsgen.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_PATH):
            raise ImportError(f"{_PATH} missing: run python -m paper_2111_04289_b200.build")
        _lib = C.CDLL(_PATH)
        _lib.lmsgen_lr_second.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                          C.c_void_p, C.c_void_p]
        _lib.lmsgen_lr_second.restype = C.c_int
        _lib.lmsgen_cm_second.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int64,
                                          C.c_void_p, C.POINTER(C.c_uint64), C.c_void_p]
        _lib.lmsgen_cm_second.restype = C.c_int
    return _lib


def gen_second(family: str, t: int, count: int, out_ptr: int, seed: int = SEED, params=None,
               stream: int = 0) -> int:
    """Write second t's `count` records to device pointer out_ptr; return the byte count."""
    if family == "LR":
        p = params or LRParams()
        st = lib().lmsgen_lr_second(seed, t, count, p.num_xways, p.num_vehicles, C.c_void_p(out_ptr),
                                    C.c_void_p(stream))
        if st:
            raise RuntimeError(f"lmsgen_lr_second failed: cudaError {st}")
        return 70 * count
    p = params or CMParams()
    nb = C.c_uint64()
    st = lib().lmsgen_cm_second(seed, t, count, p.num_jobs, -1 if p.sel_ppm is None else p.sel_ppm,
                                C.c_void_p(out_ptr), C.byref(nb), C.c_void_p(stream))
    if st:
        raise RuntimeError(f"lmsgen_cm_second failed: cudaError {st}")
    return nb.value


def max_bytes(family: str, count: int) -> int:
    return (70 if family == "LR" else 145) * count


def second_tensor(family: str, t: int, count: int, seed: int = SEED, params=None, pad: int = 64):
    """Generate second t into a new torch CUDA uint8 tensor (trimmed view + the owning buffer)."""
    import torch
    buf = torch.empty(max_bytes(family, count) + pad, dtype=torch.uint8, device="cuda")
    n = gen_second(family, t, count, buf.data_ptr(), seed, params,
                   stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.current_stream().synchronize()
    return buf, n


def counts(traffic: str, seconds: int, seed: int = SEED, t0: int = 0):
    tr = Traffic.parse(traffic)
    return [tr.count(t, seed) for t in range(t0, t0 + seconds)]
