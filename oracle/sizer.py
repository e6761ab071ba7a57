"""Oracle: micro-batch admission — Eq. 4, 5, 6 and Algorithm 1 (TEST INFRASTRUCTURE ONLY).

PAPER.md §III-B/§III-C:
  Eq. 4  AvgThPut_i = sum_{k<=i} bytes_k / sum_{k<=i} Proc_k   (R12: the
                 inner sum over partitions is the batch byte count)
  Eq. 5  MaxLat_i = max_{j in NumDS_i} Buff_(i,j) + Proc_i
  Eq. 6  EstMaxLat_i = max_j Buff_(i,j) + sum_j Part_(i,j) / AvgThPut_{i-1}
                 (R13: the sum is the total batch bytes)
  Algorithm 1 ConstructMicroBatch: tmp = buffered U new (sorted by
  creation time); sliding (SlideTime > 0): admit iff EstMaxLat >= SlideTime;
  tumbling: admit iff EstMaxLat >= mean of past MaxLat (Eq. 3, R11);
  otherwise buffered = tmp.
SPEC.md decisions taken as readings:
  R15 bootstrap: no completed batch (no AvgThPut_{i-1}) -> admit the first
      non-empty poll;
  R11 tumbling with < 2 completed batches -> admit, then the mean over
      all completed batches;
  R22 "no new data" returns (False) only when buffered and new are both empty
      (S:189), so buffered data is re-judged every 10 ms poll;
  4096-dataset cap admits immediately.
Deadline systems of the earlier revision (P:6): CG(dN), N > 0, is Algorithm 1's
sliding branch with SlideTime := N; CG(d0) is the tumbling branch (R16).
OS(tN) (P:6): admit everything buffered at every trigger instant
N, 2N, ... (if a batch overran, at the first poll after it).
"""
from __future__ import annotations

from dataclasses import dataclass, field

CAP_DATASETS = 4096


@dataclass(frozen=True)
class Dataset:
    id: int
    ingest_time: float
    nbytes: int


def est_max_lat(now: float, datasets, avg_thput_prev: float) -> float:
    """Eq. 6: max_j (now - ingest_j) + (sum_j bytes_j) / AvgThPut_{i-1}."""
    if not datasets:
        raise ValueError("empty micro-batch")
    if avg_thput_prev <= 0:
        raise ValueError("AvgThPut_{i-1} must be positive")
    max_buff = max(now - d.ingest_time for d in datasets)
    total = sum(d.nbytes for d in datasets)
    return max_buff + total / avg_thput_prev


def seq_sum(xs) -> float:
    """Plain left-to-right fp64 sum in batch order (reading R28).  Not Python's sum(): since
    3.12 that is a compensated (Neumaier) sum, a different rounding from the online running
    sum the method keeps, and an admission decision (EstMaxLat >= target) compares values
    that can differ in the last bit."""
    s = 0.0
    for x in xs:
        s += x
    return s


def avg_thput(batch_bytes: list[int], procs: list[float]) -> float:
    """Eq. 4 over batches 0..i."""
    return sum(batch_bytes) / seq_sum(procs)


def max_lat(max_buff: float, proc: float) -> float:
    """Eq. 5."""
    return max_buff + proc


@dataclass
class Decision:
    admitted: bool
    batch: list = field(default_factory=list)
    carried: list = field(default_factory=list)
    est_max_lat: float | None = None
    reason: str = ""


def construct_micro_batch(buffered, new_files, now: float, *, mode: str, slide_s: float,
                          deadline_s: float, avg_thput_prev: float | None,
                          max_lat_history: list[float]) -> Decision:
    """Algorithm 1 for mode in {"lmstream", "deadline"}.

    slide_s: SlideTime of the query (0 = tumbling); deadline_s: CG(dN)'s N.
    """
    if not buffered and not new_files:
        return Decision(False, reason="poll")
    tmp = list(buffered) + sorted(new_files, key=lambda d: (d.ingest_time, d.id))
    if len(tmp) >= CAP_DATASETS:
        return Decision(True, tmp, reason="cap")
    if avg_thput_prev is None or avg_thput_prev <= 0:
        return Decision(True, tmp, reason="bootstrap")
    est = est_max_lat(now, tmp, avg_thput_prev)
    if mode == "lmstream":
        sliding, target = slide_s > 0, slide_s
    elif mode == "deadline":
        sliding, target = deadline_s > 0, deadline_s
    else:
        raise ValueError(mode)
    if sliding:
        if est >= target:
            return Decision(True, tmp, est_max_lat=est, reason="slide")
    else:
        if len(max_lat_history) < 2:
            return Decision(True, tmp, est_max_lat=est, reason="tumbling-bootstrap")
        mean = seq_sum(max_lat_history) / len(max_lat_history)
        if est >= mean:
            return Decision(True, tmp, est_max_lat=est, reason="tumbling")
    return Decision(False, carried=tmp, est_max_lat=est, reason="buffer")


class Admission:
    """Stateful Algorithm 1 driver over a virtual clock (one batch in flight at a time)."""

    def __init__(self, mode: str, slide_s: float = 0.0, deadline_s: float = 0.0,
                 trigger_s: float = 0.0):
        self.mode, self.slide_s, self.deadline_s, self.trigger_s = mode, slide_s, deadline_s, trigger_s
        self.buffered = []
        self.pending_new = []
        self.bytes_hist, self.proc_hist, self.maxlat_hist = [], [], []
        self.next_trigger = trigger_s
        self.in_flight = None

    @property
    def avg_thput(self):
        return avg_thput(self.bytes_hist, self.proc_hist) if self.proc_hist else None

    def push(self, d: Dataset):
        self.pending_new.append(d)

    def poll(self, now: float) -> Decision:
        if self.in_flight is not None:
            return Decision(False, reason="in-flight")
        new, self.pending_new = self.pending_new, []
        if self.mode == "trigger":
            tmp = list(self.buffered) + sorted(new, key=lambda d: (d.ingest_time, d.id))
            if now >= self.next_trigger:
                self.next_trigger = (now // self.trigger_s + 1) * self.trigger_s
                if tmp:
                    self.buffered = []
                    return self._admit(Decision(True, tmp, reason="trigger"), now)
            self.buffered = tmp
            return Decision(False, carried=tmp, reason="trigger-wait")
        if self.mode == "manual":
            self.buffered = list(self.buffered) + new
            return Decision(False, carried=self.buffered, reason="manual")
        d = construct_micro_batch(self.buffered, new, now, mode=self.mode, slide_s=self.slide_s,
                                  deadline_s=self.deadline_s, avg_thput_prev=self.avg_thput,
                                  max_lat_history=self.maxlat_hist)
        if d.admitted:
            self.buffered = []
            return self._admit(d, now)
        self.buffered = d.carried
        return d

    def force(self, now: float) -> Decision:
        tmp = list(self.buffered) + sorted(self.pending_new, key=lambda d: (d.ingest_time, d.id))
        self.buffered, self.pending_new = [], []
        if not tmp:
            return Decision(False, reason="empty")
        return self._admit(Decision(True, tmp, reason="forced"), now)

    def _admit(self, d: Decision, now: float) -> Decision:
        self.in_flight = (now, d.batch)
        return d

    def complete(self, proc: float):
        """Batch finished after proc seconds: update Eq. 4 / Eq. 5 history."""
        now, batch = self.in_flight
        self.in_flight = None
        mb = max(now - x.ingest_time for x in batch)
        self.bytes_hist.append(sum(x.nbytes for x in batch))
        self.proc_hist.append(proc)
        self.maxlat_hist.append(max_lat(mb, proc))
        return self.maxlat_hist[-1]
