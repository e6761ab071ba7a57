"""Column form of the lmsgen draws, vectorised with numpy (INPUT GENERATION ONLY).

The same counter-based SplitMix64 draws as lmsgen/__init__.py, for a
whole second of records at once: field values as numpy arrays instead of formatted bytes.
Used by the full-size (10M records per batch) parity tests, whose oracle side
(oracle/bulk.py) aggregates these columns, while the CUDA path parses the byte stream that
lmsgen/gen.cu produces from the same draws.  Pinned to the scalar generator by
tests/test_oracle_gen.py.  Holds none of the method's arithmetic.
"""
from __future__ import annotations

import numpy as np

from . import (CM_EVENT_THRESHOLDS, SEED, TAG_CM, TAG_KEY, TAG_LR, CMParams, LRParams, _mu, _sec_prefix, r)

_C1 = np.uint64(0x9E3779B97F4A7C15)
_C2 = np.uint64(0xBF58476D1CE4E5B9)
_C3 = np.uint64(0x94D049BB133111EB)
_M32 = np.uint64(0xFFFFFFFF)


def mix(z: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser on a uint64 array (wrap-around arithmetic)."""
    with np.errstate(over="ignore"):
        z = z + _C1
        z = (z ^ (z >> np.uint64(30))) * _C2
        z = (z ^ (z >> np.uint64(27))) * _C3
        return z ^ (z >> np.uint64(31))


def u(x: np.ndarray, n: int) -> np.ndarray:
    """floor(x * n / 2^64) for uint64 x and 0 < n < 2^64 (128-bit product from 32-bit limbs)."""
    n = int(n)
    a, b = x >> np.uint64(32), x & _M32
    c, d = np.uint64(n >> 32), np.uint64(n & 0xFFFFFFFF)
    with np.errstate(over="ignore"):
        bd_hi = (b * d) >> np.uint64(32)
        m1 = a * d + bd_hi
        m2 = b * c + (m1 & _M32)
        return a * c + (m1 >> np.uint64(32)) + (m2 >> np.uint64(32))


def _prefix(seed: int, tag: int, t: int, count: int) -> np.ndarray:
    """Per-record prefix mix(mix(mix(mix(seed) ^ tag) ^ t) ^ i), i = 0 .. count-1."""
    return mix(np.uint64(_sec_prefix(seed, tag, t)) ^ np.arange(count, dtype=np.uint64))


def _draw(p: np.ndarray, f: int) -> np.ndarray:
    return mix(p ^ np.uint64(f))


def lr_columns(seed: int, t: int, count: int, p: LRParams = LRParams()) -> dict:
    """LR field columns of second t (lmsgen.lr_fields for i = 0 .. count-1)."""
    pre = _prefix(seed, TAG_LR, t, count)
    xway = u(_draw(pre, 1), p.num_xways).astype(np.int64)
    d = u(_draw(pre, 2), 2).astype(np.int64)
    seg = u(_draw(pre, 3), 100).astype(np.int64)
    k = (xway * 2 + d) * 100 + seg
    mu = np.array([_mu(seed, kk) for kk in range(200 * p.num_xways)], dtype=np.int64)
    spd = np.clip(mu[k] + u(_draw(pre, 5), 21).astype(np.int64) - 10, 0, 100)
    return dict(ts=np.full(count, t, dtype=np.int64), vid=u(_draw(pre, 0), p.num_vehicles).astype(np.int64),
                xway=xway, dir=d, seg=seg, lane=u(_draw(pre, 4), 5).astype(np.int64), spd=spd)


def cm_columns(seed: int, t: int, count: int, p: CMParams = CMParams()) -> dict:
    """CM field columns of second t (lmsgen.cm_fields for i = 0 .. count-1): ts, jobId,
    eventType, category, cpu * 10^6."""
    pre = _prefix(seed, TAG_CM, t, count)
    j = u(_draw(pre, 1), p.num_jobs).astype(np.int64)
    jobs = np.array([10 ** 9 + ((r(seed, TAG_KEY, 0, jj, 1) * 9 * 10 ** 9) >> 64) for jj in range(p.num_jobs)],
                    dtype=np.uint64)
    if p.sel_ppm is None:
        e = u(_draw(pre, 4), 100).astype(np.int64)
        ev = np.searchsorted(np.array(CM_EVENT_THRESHOLDS), e, side="right")
    else:
        hit = u(_draw(pre, 4), 10 ** 6).astype(np.int64) < p.sel_ppm
        other = np.array((0, 2, 3, 4, 5, 6, 7, 8))[u(_draw(pre, 11), 8).astype(np.int64)]
        ev = np.where(hit, 1, other)
    return dict(ts=np.full(count, t, dtype=np.int64), job=jobs[j], event=ev.astype(np.int64),
                cat=u(_draw(pre, 5), 4).astype(np.int64), cpu_m=1 + u(_draw(pre, 7), 500000).astype(np.int64))


__all__ = ["mix", "u", "lr_columns", "cm_columns", "SEED"]
