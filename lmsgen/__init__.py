"""lmsgen — seeded synthetic input generators for the LMStream hot path.

This module is INPUT GENERATION ONLY.  It holds none of the method's
arithmetic (no framing, parsing, filtering, windowing or aggregation): it
draws field values and formats record bytes.  It is the one module that both
the oracle (``oracle/``) and the CUDA path's tests / bench may use, so the two
sides are checked on identical bytes.

What it generates (PAPER.md = /root/reference/PAPER.md, line P:n):

* Traffic families of the paper's earlier revision:
  B(N) "a constant number of (N*1000) records every second",
  U(N) "a random record that converges to a specific average value (N*1000)",
  R(L,U) "a random record with a lower limit (L*1000) and an upper limit (U*1000)".
  The final paper's "constant" traffic (1000 rows/s) is B(1); its
  "random" traffic "normal distribution of 1000 as an average point"
  is read as U(1) with an integer Irwin-Hall normal, sigma = mean/4
  (SPEC.md S:127 default; reading R10).
* Record formats: Linear Road "70 B (per record, fixed)" and Cluster
  Monitoring "130 ~ 145 B (per record, variable)"; field names
  from Table IV.  The byte layouts are our
  reading (R1), fixed in SURVEY.md Appendix A.

All draws are integer-only counter-based SplitMix64 (no libm, no platform
RNG), so the CUDA generator in ``lmsgen/gen.cu`` reproduces these bytes
exactly; tests pin that equality and golden SHA-256 digests
(``tests/golden/gen_*.sha256``).
"""
from __future__ import annotations

import functools
import re
from dataclasses import dataclass

M64 = (1 << 64) - 1
SEED = 211104289

TAG_LR = 1
TAG_CM = 2
TAG_COUNT = 3
TAG_KEY = 4

LR_RECORD_BYTES = 70
B64 = b"ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/"
CM_EVENT_THRESHOLDS = (26, 52, 54, 56, 78, 96, 97, 99, 100)


def mix(z: int) -> int:
    """SplitMix64 finaliser (one step)."""
    z = (z + 0x9E3779B97F4A7C15) & M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def r(seed: int, tag: int, t: int, i: int, f: int) -> int:
    """Counter-based draw r(seed, tag, t, i, f)."""
    return mix(mix(mix(mix(mix(seed) ^ tag) ^ t) ^ i) ^ f)


@functools.lru_cache(maxsize=4096)
def _sec_prefix(seed: int, tag: int, t: int) -> int:
    return mix(mix(mix(seed) ^ tag) ^ t)


class _Rec:
    """r(seed, tag, t, i, f) for a fixed record (seed, tag, t, i): one mix per draw."""

    __slots__ = ("p",)

    def __init__(self, seed: int, tag: int, t: int, i: int):
        self.p = mix(_sec_prefix(seed, tag, t) ^ i)

    def __call__(self, f: int) -> int:
        return mix(self.p ^ f)


def u(x: int, n: int) -> int:
    """Map a 64-bit draw to [0, n): the high 64 bits of the 128-bit product."""
    return (x * n) >> 64


# --------------------------------------------------------------------------- traffic

@dataclass(frozen=True)
class Traffic:
    """Per-second record counts c_t.  kind in {"B", "U", "R"}; rates in records/s."""

    kind: str
    rate: int = 0       # B, U: rho = N*1000
    lo: int = 0         # R: L*1000
    hi: int = 0         # R: U*1000

    @staticmethod
    def parse(spec: str) -> "Traffic":
        m = re.fullmatch(r"\s*([BUR])\(\s*([0-9.]+)\s*(?:,\s*([0-9.]+)\s*)?\)\s*", spec)
        if not m:
            raise ValueError(f"bad traffic spec {spec!r}")
        kind = m.group(1)

        def k1000(s: str) -> int:
            v = round(float(s) * 1000)
            if abs(v - float(s) * 1000) > 1e-6:
                raise ValueError(f"N*1000 must be an integer in {spec!r}")
            return v

        if kind == "R":
            if m.group(3) is None:
                raise ValueError(spec)
            lo, hi = k1000(m.group(2)), k1000(m.group(3))
            if not (0 < lo <= hi):
                raise ValueError(spec)
            return Traffic("R", lo=lo, hi=hi)
        if m.group(3) is not None:
            raise ValueError(spec)
        rate = k1000(m.group(2))
        if rate <= 0:
            raise ValueError(spec)
        return Traffic(kind, rate=rate)

    def count(self, t: int, seed: int = SEED) -> int:
        """Records generated in second t."""
        if self.kind == "B":
            return self.rate
        if self.kind == "R":
            return self.lo + u(_Rec(seed, TAG_COUNT, t, 0)(0), self.hi - self.lo + 1)
        # U: Irwin-Hall(12) normal in integer arithmetic, sigma = rate // 4.
        rr = _Rec(seed, TAG_COUNT, t, 0)
        s = sum(rr(k) >> 32 for k in range(1, 13))
        sigma = self.rate // 4
        return max(1, self.rate + (sigma * (s - 6 * (1 << 32))) // (1 << 32))


# --------------------------------------------------------------------------- records

@dataclass(frozen=True)
class LRParams:
    num_xways: int = 10          # H
    num_vehicles: int = 10 ** 6  # V


@dataclass(frozen=True)
class CMParams:
    num_jobs: int = 10 ** 4      # J
    sel_ppm: int | None = None   # eventType==1 selectivity sweep (None: default mix, 0.26)


@functools.lru_cache(maxsize=None)
def _mu(seed: int, k: int) -> int:
    return 10 + u(r(seed, TAG_KEY, 0, k, 0), 81)


def lr_fields(seed: int, t: int, i: int, p: LRParams = LRParams()) -> dict:
    """Field values of LR record i of second t."""
    rr = _Rec(seed, TAG_LR, t, i)
    vid = u(rr(0), p.num_vehicles)
    xway = u(rr(1), p.num_xways)
    d = u(rr(2), 2)
    seg = u(rr(3), 100)
    lane = u(rr(4), 5)
    k = (xway * 2 + d) * 100 + seg
    spd = _mu(seed, k) + u(rr(5), 21) - 10
    spd = min(100, max(0, spd))
    pos = seg * 5280 + u(rr(6), 5280)
    return dict(type=0, time=t, vid=vid, spd=spd, xway=xway, lane=lane, dir=d, seg=seg, pos=pos,
                qid=0, sinit=0, send=0, dow=0, tod=0, day=0)


def lr_format(f: dict) -> bytes:
    s = (f"{f['type']:01d},{f['time']:06d},{f['vid']:010d},{f['spd']:03d},{f['xway']:03d},"
         f"{f['lane']:01d},{f['dir']:01d},{f['seg']:03d},{f['pos']:08d},{f['qid']:08d},"
         f"{f['sinit']:02d},{f['send']:02d},{f['dow']:01d},{f['tod']:04d},{f['day']:02d}\n")
    b = s.encode()
    assert len(b) == LR_RECORD_BYTES, (len(b), s)
    return b


def lr_record(seed: int, t: int, i: int, p: LRParams = LRParams()) -> bytes:
    return lr_format(lr_fields(seed, t, i, p))


def cm_fields(seed: int, t: int, i: int, p: CMParams = CMParams()) -> dict:
    """Field values of CM record i of second t."""
    rr = _Rec(seed, TAG_CM, t, i)
    L = 130 + u(rr(0), 16)
    j = u(rr(1), p.num_jobs)
    job = 10 ** 9 + u(r(seed, TAG_KEY, 0, j, 1), 9 * 10 ** 9)
    task = u(rr(2), 10 ** 4)
    machine = 1 + u(rr(3), 6 * 10 ** 9)
    if p.sel_ppm is None:
        e = u(rr(4), 100)
        ev = next(k for k, thr in enumerate(CM_EVENT_THRESHOLDS) if e < thr)
    else:
        if u(rr(4), 10 ** 6) < p.sel_ppm:
            ev = 1
        else:
            ev = (0, 2, 3, 4, 5, 6, 7, 8)[u(rr(11), 8)]
    cat = u(rr(5), 4)
    prio = u(rr(6), 12)
    cpu = 1 + u(rr(7), 500000)
    ram = 1 + u(rr(8), 500000)
    disk = 1 + u(rr(9), 500000)
    cons = u(rr(10), 2)
    return dict(len=L, ts=t, job=job, task=task, machine=machine, event=ev, cat=cat, prio=prio,
                cpu_m=cpu, ram_m=ram, disk_m=disk, cons=cons)


def cm_format(seed: int, t: int, i: int, f: dict) -> bytes:
    head = f"{f['ts']},,{f['job']},{f['task']},{f['machine']},{f['event']},".encode()
    tail = (f",{f['cat']},{f['prio']},0.{f['cpu_m']:06d},0.{f['ram_m']:06d},"
            f"0.{f['disk_m']:06d},{f['cons']}\n").encode()
    ulen = f["len"] - len(head) - len(tail)
    if ulen < 1:
        raise ValueError("record fields exceed the drawn length")  # cannot happen for ts < 10**9
    rr = _Rec(seed, TAG_CM, t, i)
    user = bytes(B64[u(rr(16 + c), 64)] for c in range(ulen))
    b = head + user + tail
    assert len(b) == f["len"]
    return b


def cm_record(seed: int, t: int, i: int, p: CMParams = CMParams()) -> bytes:
    return cm_format(seed, t, i, cm_fields(seed, t, i, p))


# --------------------------------------------------------------------------- datasets

def second_bytes(family: str, t: int, count: int, seed: int = SEED, params=None) -> bytes:
    """All records of second t (one dataset, ingest time t) concatenated."""
    if family == "LR":
        p = params or LRParams()
        return b"".join(lr_record(seed, t, i, p) for i in range(count))
    if family == "CM":
        p = params or CMParams()
        return b"".join(cm_record(seed, t, i, p) for i in range(count))
    raise ValueError(family)


def stream_datasets(family: str, traffic: Traffic | str, seconds: int, seed: int = SEED,
                    params=None, t0: int = 0):
    """Yield (t, bytes) for seconds t0 .. t0+seconds-1 (one dataset per second)."""
    tr = Traffic.parse(traffic) if isinstance(traffic, str) else traffic
    for t in range(t0, t0 + seconds):
        yield t, second_bytes(family, t, tr.count(t, seed), seed, params)


def family_of(query: str) -> str:
    q = query.upper()
    if q.startswith("LR"):
        return "LR"
    if q.startswith("CM"):
        return "CM"
    raise ValueError(query)
