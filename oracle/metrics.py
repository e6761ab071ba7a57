"""Oracle: latency statistics (TEST INFRASTRUCTURE ONLY).

p-th percentile by nearest rank: sort ascending, take the
value at rank ceil(p/100 * n) (1-based).  Tail latency of batch i is MaxLat_i
(Eq. 5); average latency is the mean over datasets of completion minus
ingest time (reading R17; the paper references but never prints the
"average/tail latency" equations).
"""
from __future__ import annotations

from fractions import Fraction


def percentile_nearest_rank(values, p: float) -> float:
    v = sorted(values)
    if not v:
        raise ValueError("empty")
    n = len(v)
    rank = -(-Fraction(p) * n // 100)          # ceil(p*n/100) exactly
    rank = max(1, int(rank))
    return v[rank - 1]


def avg_dataset_latency(completions: list[tuple[float, float]]) -> float:
    """completions: (ingest_time, completion_time) per dataset."""
    return sum(c - i for i, c in completions) / len(completions)
