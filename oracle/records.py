"""Oracle: record framing, field decode and validation (TEST INFRASTRUCTURE ONLY).

The paper gives only record sizes — Linear Road "70 B (per record, fixed)",
Cluster Monitoring "130 ~ 145 B (per record, variable)" (PAPER.md P:22, P:28,
rev-A Table) — the operator "Scan (CSV File)" (Table III) and the
field names of SegSpeedStr / TaskEvents (Table IV, P:897, P:903, P:910,
P:915).  The byte grammar below is our reading R1, fixed in
SURVEY.md §8c step 2 and Appendix A.  A record violating it is "bad": it is
counted and dropped (reading R21).

LR record (exactly 70 bytes, fixed-width CSV, zero-padded digits):
  Type(1),Time(6),VID(10),Spd(3),XWay(3),Lane(1),Dir(1),Seg(3),Pos(8),QID(8),
  Sinit(2),Send(2),DOW(1),TOD(4),Day(2)\\n
  valid iff: byte 69 == '\\n'; bytes at LR_COMMAS == ','; every other byte is
  an ASCII digit; Dir <= 1; Seg <= 99; XWay < num_xways (Linear Road domains).

CM record (one '\\n'-terminated CSV line, 13 columns, Google task_events order):
  ts,missing,jobId,taskIndex,machineId,eventType,user,category,priority,cpu,ram,disk,constraint
  valid iff: the line (without '\\n') is at most 255 bytes and was
  '\\n'-terminated; exactly 13 comma-separated fields; ts = 1..9 digits; missing is
  empty; jobId = 1..19 digits; eventType = 1 digit; category = 1 digit;
  cpu = D.DDDDDD (one digit, '.', six digits).  Other fields are free text
  without ',' or '\\n'.
  cpu value = cpu_m / 10**6 in fp64 (correctly rounded), cpu_m the integer
  D*10**6 + DDDDDD (reading R20: equal to float(text)).
"""
from __future__ import annotations

from dataclasses import dataclass

LR_BYTES = 70
LR_COMMAS = (1, 8, 19, 23, 27, 29, 31, 35, 44, 53, 56, 59, 61, 66)
LR_NEWLINE = 69
# (name, start, end) byte ranges of the decoded LR fields
LR_FIELDS = {
    "time": (2, 8), "vid": (9, 19), "spd": (20, 23), "xway": (24, 27),
    "lane": (28, 29), "dir": (30, 31), "seg": (32, 35),
}
DIGITS = b"0123456789"
CM_MAX_LINE = 255          # bytes before the '\n' (reading R1: longer lines are malformed)


@dataclass(frozen=True)
class LRRecord:
    ts: int
    vehicle: int
    speed: int
    xway: int
    lane: int
    dir: int
    seg: int


@dataclass(frozen=True)
class CMRecord:
    ts: int
    job: int
    event: int
    cat: int
    cpu_m: int       # cpu * 10**6, exact integer

    @property
    def cpu(self) -> float:
        return self.cpu_m / 10 ** 6


def parse_lr_record(rec: bytes, num_xways: int = 10):
    """Decode one 70-byte LR record; return LRRecord or None if invalid."""
    if len(rec) != LR_BYTES:
        return None
    if rec[LR_NEWLINE] != ord("\n"):
        return None
    for pos in range(LR_NEWLINE):
        c = rec[pos]
        if pos in LR_COMMAS:
            if c != ord(","):
                return None
        elif c not in DIGITS:
            return None

    def fld(name):
        a, b = LR_FIELDS[name]
        return int(rec[a:b].decode())

    r = LRRecord(ts=fld("time"), vehicle=fld("vid"), speed=fld("spd"), xway=fld("xway"),
                 lane=fld("lane"), dir=fld("dir"), seg=fld("seg"))
    if r.dir > 1 or r.seg > 99 or r.xway >= num_xways:
        return None
    return r


def frame_lr(data: bytes) -> list[bytes]:
    """Fixed-width framing: record i is data[70 i : 70 i + 70]."""
    if len(data) % LR_BYTES:
        raise ValueError("LR dataset length is not a multiple of 70")
    return [data[i:i + LR_BYTES] for i in range(0, len(data), LR_BYTES)]


def _digits(s: bytes, lo: int, hi: int) -> bool:
    return lo <= len(s) <= hi and all(c in DIGITS for c in s)


def parse_cm_record(line: bytes):
    """Decode one CM line (without its '\\n'); return CMRecord or None if invalid."""
    if len(line) > CM_MAX_LINE:
        return None
    f = line.split(b",")
    if len(f) != 13:
        return None
    if not _digits(f[0], 1, 9):
        return None
    if f[1] != b"":
        return None
    if not _digits(f[2], 1, 19):
        return None
    if not _digits(f[5], 1, 1) or not _digits(f[7], 1, 1):
        return None
    cpu = f[9]
    if len(cpu) != 8 or cpu[1] != ord(".") or not _digits(cpu[:1], 1, 1) or not _digits(cpu[2:], 6, 6):
        return None
    cpu_m = int(cpu[:1].decode()) * 10 ** 6 + int(cpu[2:].decode())
    return CMRecord(ts=int(f[0].decode()), job=int(f[2].decode()), event=int(f[5].decode()),
                    cat=int(f[7].decode()), cpu_m=cpu_m)


def frame_cm(data: bytes) -> tuple[list[bytes], int]:
    """Newline framing: the records are the '\\n'-terminated lines of the dataset.

    Returns (lines, n_unterminated): bytes after the last '\\n' form one
    unterminated (hence malformed) record.
    """
    lines = data.split(b"\n")
    tail = lines.pop()
    return lines, (1 if tail else 0)


def parse_dataset(family: str, data: bytes, num_xways: int = 10):
    """Return (records_in_order, n_bad) for one dataset."""
    out, bad = [], 0
    if family == "LR":
        for rec in frame_lr(data):
            r = parse_lr_record(rec, num_xways)
            if r is None:
                bad += 1
            else:
                out.append(r)
    elif family == "CM":
        lines, unterminated = frame_cm(data)
        bad += unterminated
        for line in lines:
            r = parse_cm_record(line)
            if r is None:
                bad += 1
            else:
                out.append(r)
    else:
        raise ValueError(family)
    return out, bad
