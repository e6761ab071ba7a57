"""Pins for oracle/records.py: the record grammar (reading R1) by example."""
import random

import lmsgen as g
from oracle import records as R


def lr_bytes(**kw):
    f = dict(type=0, time=0, vid=0, spd=0, xway=0, lane=0, dir=0, seg=0, pos=0, qid=0,
             sinit=0, send=0, dow=0, tod=0, day=0)
    f.update(kw)
    return g.lr_format(f)


def test_lr_field_offsets_by_hand():
    b = b"0,000123,0000000042,055,003,2,1,077,00406560,00000000,00,00,0,0000,00\n"
    assert len(b) == 70
    r = R.parse_lr_record(b)
    assert (r.ts, r.vehicle, r.speed, r.xway, r.lane, r.dir, r.seg) == (123, 42, 55, 3, 2, 1, 77)


def test_lr_every_separator_and_digit_is_checked():
    good = lr_bytes(time=5, vid=99, spd=31, xway=2, seg=14)
    assert R.parse_lr_record(good) is not None
    for pos in range(70):
        bad = bytearray(good)
        bad[pos] = ord("a")                      # not a digit, not a separator
        assert R.parse_lr_record(bytes(bad)) is None, pos
    for pos in R.LR_COMMAS:
        bad = bytearray(good)
        bad[pos] = ord("7")
        assert R.parse_lr_record(bytes(bad)) is None
    bad = bytearray(good)
    bad[69] = ord(",")
    assert R.parse_lr_record(bytes(bad)) is None


def test_lr_domains():
    assert R.parse_lr_record(lr_bytes(dir=2)) is None
    assert R.parse_lr_record(lr_bytes(seg=100)) is None
    assert R.parse_lr_record(lr_bytes(xway=10)) is None
    assert R.parse_lr_record(lr_bytes(xway=10), num_xways=11) is not None
    assert R.parse_lr_record(lr_bytes(xway=9, dir=1, seg=99, spd=999)) is not None


def test_cm_grammar_examples():
    ok = b"17,,5727399796,7831,5426611511,1,U9kE,3,0,0.294913,0.368826,0.097151,1"
    r = R.parse_cm_record(ok)
    assert (r.ts, r.job, r.event, r.cat, r.cpu_m) == (17, 5727399796, 1, 3, 294913)
    assert r.cpu == 0.294913
    bad = [
        b"17,,5727399796,7831,5426611511,1,U9kE,3,0,0.294913,0.368826,0.097151",       # 12 fields
        b"17,,5727399796,7831,5426611511,1,U9kE,3,0,0.294913,0.368826,0.097151,1,9",   # 14 fields
        b",,5727399796,7831,5426611511,1,U9kE,3,0,0.294913,0.368826,0.097151,1",       # empty ts
        b"1234567890,,57,1,1,1,u,3,0,0.294913,1,1,1",                                  # ts 10 digits
        b"17,x,5727399796,7831,5426611511,1,U9kE,3,0,0.294913,0.368826,0.097151,1",    # missing not empty
        b"17,,57273997a6,7831,5426611511,1,U9kE,3,0,0.294913,0.368826,0.097151,1",     # job non digit
        b"17,,12345678901234567890,1,1,1,u,3,0,0.294913,1,1,1",                        # job 20 digits
        b"17,,5727399796,7831,5426611511,11,U9kE,3,0,0.294913,0.368826,0.097151,1",    # event 2 digits
        b"17,,5727399796,7831,5426611511,1,U9kE,,0,0.294913,0.368826,0.097151,1",      # empty category
        b"17,,5727399796,7831,5426611511,1,U9kE,3,0,0.29491,0.368826,0.097151,1",      # cpu 5 frac digits
        b"17,,5727399796,7831,5426611511,1,U9kE,3,0,0,294913,0.368826,0.097151,1",     # cpu comma
        b"17,,5727399796,7831,5426611511,1,U9kE,3,0,10.29491,0.368826,0.097151,1",     # cpu 2 int digits
        b"",
    ]
    for b in bad:
        assert R.parse_cm_record(b) is None, b
    assert R.parse_cm_record(b"1,,1,,,0,,0,,9.999999,,,") is not None   # free fields may be empty


def test_cm_cpu_equals_float_of_text():
    rng = random.Random(5)
    for _ in range(20000):
        m = rng.randrange(0, 10 ** 7)
        text = f"{m // 10 ** 6}.{m % 10 ** 6:06d}"
        line = f"1,,2,3,4,1,u,0,0,{text},0,0,0".encode()
        assert R.parse_cm_record(line).cpu == float(text)


def test_framing():
    data = b"".join(g.cm_record(g.SEED, 0, i) for i in range(10))
    lines, unterminated = R.frame_cm(data)
    assert unterminated == 0
    assert len(lines) == 10 and all(not ln.endswith(b"\n") for ln in lines)
    recs, bad = R.parse_dataset("CM", data)
    assert len(recs) == 10 and bad == 0
    data = b"".join(g.lr_record(g.SEED, 0, i) for i in range(10))
    recs, bad = R.parse_dataset("LR", data)
    assert len(recs) == 10 and bad == 0
    recs, bad = R.parse_dataset("CM", b"garbage\n" + g.cm_record(g.SEED, 0, 1) + b"\n")
    assert len(recs) == 1 and bad == 2


def test_cm_line_length_limit_and_unterminated_tail():
    base = b"1,,2,3,4,1,,0,0,0.000001,0,0,"
    assert R.parse_cm_record(base + b"1" * (255 - len(base))) is not None
    assert R.parse_cm_record(base + b"1" * (256 - len(base))) is None
    recs, bad = R.parse_dataset("CM", g.cm_record(g.SEED, 0, 0) + b"1,,2,3,4,1,,0,0,0.000001,0,0,0")
    assert len(recs) == 1 and bad == 1
