"""Virtual-clock driver of the LMStream micro-batch loop (host control only).

PAPER.md §III-C: the stream engine checks for new datasets every 10 ms and calls
ConstructMicroBatch (Alg. 1) — `lms_poll` here; one micro-batch is in flight at
a time (a batch is admitted only after the previous one completed).  Configs C2/C3/C5
(BASELINE.json) run minutes of stream time; this driver replays them on a VIRTUAL clock:
datasets become visible at their ingest time, a poll happens every `poll_s` of virtual time,
and an admitted batch is run for real on the GPU — its measured Proc (lms_batch_record.proc_s:
device time + result D2H, reading R18) advances the virtual clock to the first poll tick at
or after admit_time + Proc.  Eq. 5 latencies are therefore those of a real-time run without
waiting the real seconds (SURVEY §8d "virtual s").

Every batch runs through the C ABI (`lms_poll` / `lms_sync` / `lms_flush`); this module only
sequences calls.  The oracle mirror of the same loop lives in tests/test_gpu_sizer.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

from ._lib import LMS_EFORMAT, LMS_OK


@dataclass
class Arrival:
    ingest_s: float
    data: object                 # bytes / numpy uint8 / (host ptr, nbytes) / ("dev", ptr, nbytes)
    nbytes: int


@dataclass
class SimResult:
    records: list = field(default_factory=list)       # lms_batch_record dicts, batch order
    rows: list = field(default_factory=list)          # result rows per batch (numpy)
    batches: list = field(default_factory=list)       # arrival indices per batch
    polls: int = 0


def _push(query, a: Arrival):
    if isinstance(a.data, tuple) and len(a.data) == 3 and a.data[0] == "dev":
        query.push_device(a.data[1], a.data[2], a.ingest_s)
    else:
        query.push(a.data, a.ingest_s)


def run(query, arrivals: list[Arrival], t_end: float, poll_s: float = 0.01, flush: bool = True,
        read_rows: bool = True, ok=(LMS_OK, LMS_EFORMAT)) -> SimResult:
    """Drive `query` (LMSTREAM / DEADLINE / TRIGGER mode) over `arrivals` until `t_end`.

    Poll instants are tick * poll_s (integer ticks: no drift).  Arrivals must be sorted by
    ingest time; an arrival is pushed before the first poll at or after its ingest time.
    """
    lr1 = query.cfg.kind in (0, 1)
    res = SimResult()
    nxt = 0                       # next arrival to push
    pushed_ids = []               # arrival index per pending dataset (admission order)
    tick, last_tick = 0, int(math.floor(t_end / poll_s + 1e-9))
    while tick <= last_tick:
        now = tick * poll_s
        while nxt < len(arrivals) and arrivals[nxt].ingest_s <= now + 1e-12:
            _push(query, arrivals[nxt])
            pushed_ids.append(nxt)
            nxt += 1
        idx, _ = query.poll(now, ok=ok)
        res.polls += 1
        if idx is None:
            tick += 1
            continue
        query.sync(ok=ok)
        rec = query.record(idx)
        n = rec["num_datasets"]
        res.batches.append(pushed_ids[:n])
        del pushed_ids[:n]
        res.records.append(rec)
        if read_rows:
            res.rows.append(query.read_lr1() if lr1 else query.read_agg())
        # next poll: first tick at or after completion (one batch in flight at a time)
        tick = max(tick + 1, int(math.ceil((now + rec["proc_s"]) / poll_s - 1e-9)))
    if flush:
        while nxt < len(arrivals):
            _push(query, arrivals[nxt])
            pushed_ids.append(nxt)
            nxt += 1
        query.flush(tick * poll_s, ok=ok)
        rec = query.record(query.num_batches() - 1)
        res.batches.append(list(pushed_ids))
        res.records.append(rec)
        if read_rows:
            res.rows.append(query.read_lr1() if lr1 else query.read_agg())
    return res


def split_seconds(family: str, seconds, parts: int = 1):
    """(t, dataset bytes) per second -> arrivals; each second is cut into `parts` sub-datasets
    at record boundaries, sub-dataset j of second t ingested at t + (j + 1) / parts (the file
    is complete at the end of its slice of the second; reading R4)."""
    from .dist import split_points
    out = []
    for t, d in seconds:
        for j, (o, n) in enumerate(split_points(family, d, parts)):
            if n:
                out.append(Arrival(t + (j + 1) / parts, d[o:o + n], n))
    return out
