"""Oracle, column form: LR2 / CM1 / CM2 window aggregates and the LR1 self-join for full-size batches
(TEST INFRASTRUCTURE ONLY — imported by tests/ alone; the product never calls it).

Same definitions as oracle/queries.py — Table IV (P:903 LR2S, P:910 CM1, P:915 CM2S), window
instances [kS, kS+R) (R5), emission after each batch of every instance with end <= W and the
rest at flush (R7), exact integer sums (speed; cpu * 10^6) with AVG = SUM / COUNT in fp64
(R20) — restated over per-second group partials so that 10M-record batches can be checked in
seconds: every record of a dataset produced by lmsgen carries its second t as timestamp
(R4), so an instance's per-group COUNT and SUM are the sums over the seconds it covers of
that second's per-group COUNT and SUM (integer addition: the order does not matter).
Inputs are the field columns of lmsgen.vec (one dataset = one second); pinned against the
brute-force oracle.queries on small streams by tests/test_oracle_bulk.py.
"""
from __future__ import annotations

import numpy as np

from .queries import AggRow, QuerySpec


class BulkReplay:
    """Per-batch emission replay (R7) over per-second partial aggregates."""

    def __init__(self, q: QuerySpec):
        if q.name not in ("LR2S", "CM1S", "CM1T", "CM2S"):
            raise ValueError(q.name)
        self.q = q
        self.W = None            # watermark: max timestamp seen
        self.next_k = None       # first instance not yet emitted
        self.sec = {}            # t -> (unique keys, counts, exact sums)

    def _partial(self, cols: dict):
        name = self.q.name
        if name == "LR2S":      # GROUPBY (highway, direction, segment), AVG(speed)
            key = (cols["xway"] * 2 + cols["dir"]) * 100 + cols["seg"]
            val = cols["spd"]
        elif name == "CM2S":    # WHERE (eventType == 1) GROUPBY jobId, AVG(cpu)
            keep = cols["event"] == 1
            key, val = cols["job"][keep], cols["cpu_m"][keep]
        else:                   # CM1: GROUPBY category, SUM(cpu)
            key, val = cols["cat"], cols["cpu_m"]
        uk, inv = np.unique(key, return_inverse=True)
        cnt = np.bincount(inv, minlength=len(uk)).astype(np.int64)
        # integer sums < 2^53 are exact in the fp64 accumulator of bincount
        sm = np.bincount(inv, weights=val.astype(np.float64), minlength=len(uk))
        assert float(sm.sum()) < 2.0 ** 53
        return uk, cnt, sm.astype(np.int64)

    def _instance(self, k: int) -> list:
        q = self.q
        s, e = k * q.slide_s, k * q.slide_s + q.range_s
        parts = [self.sec[t] for t in range(s, e) if t in self.sec]
        if not parts:
            return []
        keys = np.concatenate([p[0] for p in parts])
        uk, inv = np.unique(keys, return_inverse=True)
        cnt = np.zeros(len(uk), np.int64)
        sm = np.zeros(len(uk), np.int64)
        np.add.at(cnt, inv, np.concatenate([p[1] for p in parts]))
        np.add.at(sm, inv, np.concatenate([p[2] for p in parts]))
        rows = []
        if q.name == "LR2S":
            for code, c, v in zip(uk.tolist(), cnt.tolist(), sm.tolist()):
                avg = v / c
                if c and avg < 40.0:                       # HAVING (avgSpeed < 40.0)
                    rows.append(AggRow(s, e, (code // 200, (code // 100) % 2, code % 100), c, v, float(v), avg))
        elif q.name == "CM2S":
            for job, c, v in zip(uk.tolist(), cnt.tolist(), sm.tolist()):
                if c:
                    rows.append(AggRow(s, e, (job,), c, v, v / 10 ** 6, (v / 10 ** 6) / c))
        else:                                              # ORDER BY SUM(cpu), ties by category
            grp = sorted((v, cat, c) for cat, c, v in zip(uk.tolist(), cnt.tolist(), sm.tolist()) if c)
            rows = [AggRow(s, e, (cat,), c, v, v / 10 ** 6, (v / 10 ** 6) / c, rank)
                    for rank, (v, cat, c) in enumerate(grp)]
        return rows

    def _emit_upto(self, k_last: int) -> list:
        rows = []
        while self.next_k <= k_last:
            rows.extend(self._instance(self.next_k))
            self.next_k += 1
        return rows

    def batch(self, t: int, cols: dict) -> list:
        """One micro-batch holding the single dataset of second t (columns of all its records)."""
        assert self.W is None or t >= self.W, "column replay needs in-order seconds (no late data)"
        if len(cols["ts"]):
            assert int(cols["ts"].min()) == t == int(cols["ts"].max())
            self.sec[t] = self._partial(cols)
            if self.next_k is None:
                self.next_k = (t - self.q.range_s) // self.q.slide_s + 1
            self.W = t if self.W is None else max(self.W, t)
        if self.W is None:
            return []
        return self._emit_upto((self.W - self.q.range_s) // self.q.slide_s)

    def flush(self) -> list:
        return [] if self.W is None else self._emit_upto(self.W // self.q.slide_s)


LR1_DTYPE = np.dtype([("win_start", "<i8"), ("ts", "<i8"), ("vehicle", "<i8"), ("speed", "<i8"),
                      ("xway", "<i8"), ("lane", "<i8"), ("dir", "<i8"), ("seg", "<i8"), ("m", "<i8")])


class BulkLr1Replay:
    """LR1S / LR1T (Table IV, reading R8) in column form: for window instance k, A = the
    records of [kS, kS+R), L = the records of its newest slide [kS+R-S, kS+R) (tumbling: L = A);
    one row per l in L with m = #{a in A : a.vehicle == l.vehicle}.  m is computed from the
    per-second vehicle counts: #{a in A : a.vehicle = v} = sum over the seconds t of A of
    #{records of second t with vehicle v} (every lmsgen record of dataset t has ts = t, R4).
    Emission as queries.Replay (R7): after each micro-batch, every instance with end <= W; the
    rest at flush.  Rows are returned as LR1_DTYPE arrays (compare as sorted multisets)."""

    def __init__(self, q: QuerySpec):
        if q.name not in ("LR1S", "LR1T"):
            raise ValueError(q.name)
        self.q = q
        self.W = None
        self.next_k = None
        self.cols = {}           # t -> columns of second t
        self.vc = {}             # t -> (unique vehicles, counts)

    def _instance(self, k: int) -> np.ndarray:
        q = self.q
        s, e = k * q.slide_s, k * q.slide_s + q.range_s
        secs_a = [t for t in range(s, e) if t in self.cols]
        secs_l = [t for t in range(e - q.slide_s, e) if t in self.cols]
        if not secs_l:
            return np.zeros(0, LR1_DTYPE)
        va = np.concatenate([self.vc[t][0] for t in secs_a])
        ca = np.concatenate([self.vc[t][1] for t in secs_a])
        uv, inv = np.unique(va, return_inverse=True)
        m = np.zeros(len(uv), np.int64)
        np.add.at(m, inv, ca)                     # window count per vehicle
        L = {f: np.concatenate([self.cols[t][f] for t in secs_l]) for f in ("ts", "vid", "spd", "xway",
                                                                             "lane", "dir", "seg")}
        out = np.zeros(len(L["ts"]), LR1_DTYPE)
        out["win_start"] = s
        out["ts"], out["vehicle"], out["speed"] = L["ts"], L["vid"], L["spd"]
        out["xway"], out["lane"], out["dir"], out["seg"] = L["xway"], L["lane"], L["dir"], L["seg"]
        out["m"] = m[np.searchsorted(uv, L["vid"])]      # every l is in A: its vehicle is in uv
        return out

    def _emit_upto(self, k_last: int) -> np.ndarray:
        rows = []
        while self.next_k <= k_last:
            rows.append(self._instance(self.next_k))
            self.next_k += 1
        return np.concatenate(rows) if rows else np.zeros(0, LR1_DTYPE)

    def batch(self, seconds: list) -> np.ndarray:
        """One micro-batch holding the datasets [(t, cols), ...] (in-order seconds)."""
        for t, cols in seconds:
            assert self.W is None or t > self.W, "column replay needs in-order seconds (no late data)"
            if len(cols["ts"]) == 0:
                continue
            assert int(cols["ts"].min()) == t == int(cols["ts"].max())
            self.cols[t] = cols
            self.vc[t] = np.unique(cols["vid"], return_counts=True)
            if self.next_k is None:
                self.next_k = (t - self.q.range_s) // self.q.slide_s + 1
            self.W = t if self.W is None else max(self.W, t)
        if self.W is None:
            return np.zeros(0, LR1_DTYPE)
        return self._emit_upto((self.W - self.q.range_s) // self.q.slide_s)

    def flush(self) -> np.ndarray:
        return np.zeros(0, LR1_DTYPE) if self.W is None else self._emit_upto(self.W // self.q.slide_s)
