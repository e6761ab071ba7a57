"""Oracle: Table IV queries over windows, brute force (TEST INFRASTRUCTURE ONLY).

Queries (Table IV):
  LR1S/LR1T  SELECT L.timestamp, L.vehicle, L.speed, L.highway, L.lane, L.direction, L.segment
             FROM SegSpeedStr [range 30 (slide 5)] as A, SegSpeedStr as L
             WHERE (A.vehicle == L.vehicle)
  LR2S       SELECT timestamp, highway, direction, segment, AVG(speed) as avgSpeed
             FROM SegSpeedStr [range 30 slide 10] GROUPBY (highway, direction, segment)
             HAVING (avgSpeed < 40.0)
  CM1S/CM1T  SELECT timestamp, category, SUM(cpu) as totalCpu
             FROM TaskEvents [range 60 (slide 10)] GROUPBY category ORDERBY SUM(cpu)
  CM2S       SELECT jobId, AVG(cpu) as avgCpu FROM TaskEvents [range 60 slide 5]
             WHERE (eventType == 1) GROUPBY jobId

Windows (readings R5, R6, R19 in DESIGN.md): instance k is the half-open event
time interval [k*S, k*S + R), for every integer k (negative included, Spark
`window()` alignment); tumbling (SlideTime = 0, Table I) means S = R.
A record with timestamp ts lies in the R/S instances k with
floor((ts-R)/S) < k <= floor(ts/S).  The aggregate queries' "timestamp"
output column is the instance start (R6).  Groups with no rows emit nothing.

LR1 (reading R8): per instance w, A = records of w, L = records of w's newest
slide [s+R-S, s+R) (tumbling: L = A); for every l in L one output row with l's
7 columns and the bag multiplicity m = #{a in A : a.vehicle == l.vehicle}.

Emission (reading R7): after micro-batch b the watermark W_b is the maximum
timestamp of all valid records seen so far; every not-yet-emitted instance
with end <= W_b is emitted; a record whose ts < W_{b-1} is late (counted,
dropped).  flush() emits every remaining instance that holds data.

This is the plain definition: each instance is evaluated by rescanning the
raw records whose ts falls inside it (indexed by second only to find them).
"""
from __future__ import annotations

from collections import defaultdict
from dataclasses import dataclass, field

from . import records as R


@dataclass(frozen=True)
class QuerySpec:
    name: str
    family: str      # "LR" or "CM"
    range_s: int     # R
    slide_s: int     # S (tumbling: S = R)
    tumbling: bool


# Table IV; SPEC.md S:146 (windows)
QUERIES = {
    "LR1S": QuerySpec("LR1S", "LR", 30, 5, False),
    "LR1T": QuerySpec("LR1T", "LR", 30, 30, True),
    "LR2S": QuerySpec("LR2S", "LR", 30, 10, False),
    "CM1S": QuerySpec("CM1S", "CM", 60, 10, False),
    "CM1T": QuerySpec("CM1T", "CM", 60, 60, True),
    "CM2S": QuerySpec("CM2S", "CM", 60, 5, False),
}


def query_spec(name: str, range_s: int | None = None, slide_s: int | None = None) -> QuerySpec:
    q = QUERIES[name.upper()]
    rng = range_s if range_s else q.range_s
    if q.tumbling:
        sl = rng
    else:
        sl = slide_s if slide_s else q.slide_s
    if sl <= 0 or rng <= 0 or sl > rng or rng % sl:
        raise ValueError("window needs 0 < S <= R and S | R")
    return QuerySpec(q.name, q.family, rng, sl, q.tumbling)


def instances_of(ts: int, q: QuerySpec) -> range:
    """Window instances k with k*S <= ts < k*S + R."""
    return range((ts - q.range_s) // q.slide_s + 1, ts // q.slide_s + 1)


# --------------------------------------------------------------------------- per instance

@dataclass(frozen=True)
class AggRow:
    """One output row of LR2 / CM1 / CM2 for window instance [win_start, win_end)."""
    win_start: int
    win_end: int
    key: tuple            # LR2 (xway, dir, seg); CM1 (category,); CM2 (jobId,)
    count: int
    sum_fixed: int        # exact integer sum in field units (speed; cpu * 10**6)
    sum: float            # fp64 SUM: LR2 exact int -> float; CM sequential fp64 sum of cpu values
    avg: float            # fp64 AVG = sum / count
    rank: int = 0         # CM1: position under ORDER BY SUM(cpu) (ties by category)


@dataclass(frozen=True)
class LR1Row:
    win_start: int
    ts: int
    vehicle: int
    speed: int
    xway: int
    lane: int
    dir: int
    seg: int
    m: int                # multiplicity of l.vehicle in A


def _in(rec, lo: int, hi: int) -> bool:
    return lo <= rec.ts < hi


def eval_instance(q: QuerySpec, recs, k: int) -> list:
    """Evaluate query q on window instance k by scanning all records."""
    s, e = k * q.slide_s, k * q.slide_s + q.range_s
    win = [x for x in recs if _in(x, s, e)]
    if q.name == "LR2S":
        groups = {}
        for x in win:
            g = groups.setdefault((x.xway, x.dir, x.seg), [0, 0])
            g[0] += x.speed
            g[1] += 1
        rows = []
        for key, (sm, cnt) in groups.items():
            avg = sm / cnt                      # Python int/int: correctly rounded fp64
            if avg < 40.0:                      # HAVING (avgSpeed < 40.0)
                rows.append(AggRow(s, e, key, cnt, sm, float(sm), avg))
        return rows
    if q.name in ("CM1S", "CM1T"):
        groups = {}
        for x in win:
            g = groups.setdefault(x.cat, [0, 0.0, 0])
            g[0] += 1
            g[1] += x.cpu                       # SUM(cpu), sequential fp64
            g[2] += x.cpu_m
        order = sorted(groups.items(), key=lambda kv: (kv[1][1], kv[0]))   # ORDER BY SUM(cpu)
        return [AggRow(s, e, (cat,), cnt, smf, sm, sm / cnt, rank)
                for rank, (cat, (cnt, sm, smf)) in enumerate(order)]
    if q.name == "CM2S":
        groups = {}
        for x in win:
            if x.event != 1:                    # WHERE (eventType == 1)
                continue
            g = groups.setdefault(x.job, [0, 0.0, 0])
            g[0] += 1
            g[1] += x.cpu
            g[2] += x.cpu_m
        return [AggRow(s, e, (job,), cnt, smf, sm, sm / cnt) for job, (cnt, sm, smf) in groups.items()]
    if q.name in ("LR1S", "LR1T"):
        newest_lo = e - q.slide_s
        A = win
        L = [x for x in win if x.ts >= newest_lo]
        rows = []
        for l in L:
            m = sum(1 for a in A if a.vehicle == l.vehicle)     # A.vehicle == L.vehicle
            rows.append(LR1Row(s, l.ts, l.vehicle, l.speed, l.xway, l.lane, l.dir, l.seg, m))
        return rows
    raise ValueError(q.name)


def brute_force_all(q: QuerySpec, recs) -> dict[int, list]:
    """Every instance that holds at least one record -> its rows (no batching)."""
    ks = set()
    for x in recs:
        ks.update(instances_of(x.ts, q))
    return {k: eval_instance(q, recs, k) for k in sorted(ks)}


# --------------------------------------------------------------------------- emission replay

@dataclass
class BatchOutput:
    rows: list = field(default_factory=list)
    n_records: int = 0      # records framed in the batch
    bad: int = 0            # malformed (dropped)
    late: int = 0           # ts < previous watermark (dropped)
    watermark: int | None = None
    windows_closed: int = 0


class Replay:
    """Per-micro-batch replay of the emission rule (reading R7).

    Keeps every kept record (plain, unbounded) and evaluates each emitted
    instance by brute force over them.
    """

    def __init__(self, q: QuerySpec, num_xways: int = 10):
        self.q = q
        self.num_xways = num_xways
        self.recs = []
        self.W = None            # watermark (max ts of kept records)
        self.next_k = None       # first instance not yet emitted

    def _emit_upto(self, k_last: int, out: BatchOutput):
        while self.next_k <= k_last:
            out.rows.extend(eval_instance(self.q, self._by_window(self.next_k), self.next_k))
            out.windows_closed += 1
            self.next_k += 1

    def _by_window(self, k):
        # index lookup only: the records whose ts is in [kS, kS+R)
        s, e = k * self.q.slide_s, k * self.q.slide_s + self.q.range_s
        out = []
        for t in range(s, e):
            out.extend(self._sec.get(t, ()))
        return out

    @property
    def _sec(self):
        if not hasattr(self, "_sec_idx"):
            self._sec_idx = defaultdict(list)
        return self._sec_idx

    def batch(self, datasets: list[bytes]) -> BatchOutput:
        out = BatchOutput()
        W_prev = self.W
        kept = []
        for d in datasets:
            recs, bad = R.parse_dataset(self.q.family, d, self.num_xways)
            out.bad += bad
            out.n_records += len(recs) + bad
            for x in recs:
                if W_prev is not None and x.ts < W_prev:
                    out.late += 1
                else:
                    kept.append(x)
        if kept:
            if self.next_k is None:
                self.next_k = min(x.ts for x in kept) - self.q.range_s
                self.next_k = self.next_k // self.q.slide_s + 1
            self.W = max([x.ts for x in kept] + ([W_prev] if W_prev is not None else []))
            for x in kept:
                self.recs.append(x)
                self._sec[x.ts].append(x)
        out.watermark = self.W
        if self.W is not None:
            # emit every instance with end <= W:  k*S + R <= W
            self._emit_upto((self.W - self.q.range_s) // self.q.slide_s, out)
        return out

    def flush(self) -> BatchOutput:
        out = BatchOutput(watermark=self.W)
        if self.W is not None:
            self._emit_upto(self.W // self.q.slide_s, out)
        return out


def replay(q: QuerySpec, batches: list[list[bytes]], num_xways: int = 10, flush: bool = True):
    """Run all batches (+ flush); return the list of BatchOutput (flush last if requested)."""
    rp = Replay(q, num_xways)
    outs = [rp.batch(b) for b in batches]
    if flush:
        outs.append(rp.flush())
    return outs
