"""Oracle: Eq. 10 online regression of the inflection point (TEST INFRASTRUCTURE ONLY).

PAPER.md §III-E: InflectionPoint = b0 + b1*Throughput + b2*Latency,
fitted after every micro-batch on the history of (average throughput, max
latency, InfPT used); target throughput = max of the history; target latency =
SlideTime (Eq. 2) or the mean of past latencies (Eq. 3).
SPEC.md readings (R24): ordinary least squares via the normal
equations; < 3 rows or a singular design -> insufficient history
(S:362); throughput regressor in MB/s; prediction clamped to
[1 KiB, 16 MiB]; default history window 256 rows.

The normal equations are solved EXACTLY in rational arithmetic (fractions of
the fp64 inputs), then rounded once to fp64.
"""
from __future__ import annotations

from fractions import Fraction

CLAMP_LO = 1024.0
CLAMP_HI = 16.0 * 1024 * 1024
MB = 1e6


def fit(rows):
    """rows: iterable of (avg_thput_Bps, max_lat_s, infpt_bytes) -> (b0, b1, b2) or None."""
    rows = list(rows)
    if len(rows) < 3:
        return None
    X = [[Fraction(1), Fraction(t / MB), Fraction(l)] for t, l, _ in rows]
    y = [Fraction(v) for _, _, v in rows]
    A = [[sum(X[r][i] * X[r][j] for r in range(len(X))) for j in range(3)] for i in range(3)]
    b = [sum(X[r][i] * y[r] for r in range(len(X))) for i in range(3)]
    # Gauss-Jordan with exact pivots
    M = [A[i] + [b[i]] for i in range(3)]
    for c in range(3):
        p = next((r for r in range(c, 3) if M[r][c] != 0), None)
        if p is None:
            return None
        M[c], M[p] = M[p], M[c]
        for r in range(3):
            if r != c and M[r][c] != 0:
                f = M[r][c] / M[c][c]
                M[r] = [M[r][k] - f * M[c][k] for k in range(4)]
    return tuple(float(M[i][3] / M[i][i]) for i in range(3))


def targets(history, slide_s: float):
    """(target throughput, target latency) from history rows (thput, lat, infpt)."""
    history = list(history)
    if not history:
        return None
    tt = max(h[0] for h in history)
    tl = slide_s if slide_s > 0 else sum(h[1] for h in history) / len(history)
    return tt, tl


def predict(betas, target_thput: float, target_lat: float) -> float:
    b0, b1, b2 = betas
    v = b0 + b1 * (target_thput / MB) + b2 * target_lat
    return min(CLAMP_HI, max(CLAMP_LO, v))
