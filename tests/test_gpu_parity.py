"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Bar (BASELINE.json north_star): keys, counts, filter results bit-exact; LR2 SUM/AVG bit-exact
(integer speed sums); CM SUM/AVG within 1e-9 relative; LR1 rows + multiplicities exact.
Inputs: seeded lmsgen streams shaped like the paper's workloads, sized so the
oracle finishes in seconds while spanning many tiles (LR tile = 512 records, CM tile = 32 KB)
with ragged tails, plus malformed / late / multi-segment / empty edge cases.
"""
import random

import pytest

import lmsgen as g
from tests.helpers import compare_run, oracle_rows, product_run

pytestmark = pytest.mark.gpu


def stream(family, traffic, seconds, seed=11, params=None, t0=0):
    return [d for _, d in g.stream_datasets(family, traffic, seconds, seed=seed, params=params, t0=t0)]


def split(secs, sizes):
    out, i = [], 0
    for s in sizes:
        out.append(secs[i:i + s])
        i += s
    if i < len(secs):
        out.append(secs[i:])
    return out


@pytest.mark.parametrize("qname,traffic,secs,bs", [
    ("LR2S", "B(1.7)", 45, [3, 7, 1, 10, 4]),      # 1700 rec/s: 4 tiles per second, ragged tail
    ("LR2S", "U(0.6)", 70, [10] * 7),
    ("CM2S", "B(1.3)", 40, [5, 5, 1, 9, 2]),       # ~180 KB/s: 6 CM tiles per second
    ("CM2S", "R(0.1,1)", 66, [5] * 13),
    ("CM1S", "B(0.9)", 75, [10, 10, 3, 20]),
    ("CM1T", "U(0.5)", 130, [30, 30, 60]),
    ("LR1S", "B(0.4)", 40, [5, 5, 2, 8]),
    ("LR1T", "B(0.3)", 65, [7, 11, 30]),
])
def test_parity_streams(qname, traffic, secs, bs):
    fam = qname[:2]
    params = g.LRParams(num_vehicles=300) if qname.startswith("LR1") else (
        g.CMParams(num_jobs=200) if fam == "CM" else None)
    data = stream(fam, traffic, secs, params=params)
    batches = split(data, bs)
    compare_run(qname, product_run(qname, batches), oracle_rows(qname, batches))


def test_lr2_single_big_batch_many_tiles():
    data = stream("LR", "B(12)", 3)                 # 36k records = 71 tiles in one batch
    batches = [data]
    compare_run("LR2S", product_run("LR2S", batches), oracle_rows("LR2S", batches))


def test_cm2_single_big_batch_many_tiles():
    data = stream("CM", "B(8)", 2)                  # 16k records ~ 2.2 MB = 67 tiles
    batches = [data]
    compare_run("CM2S", product_run("CM2S", batches), oracle_rows("CM2S", batches))


def _corrupt(data: bytes, n: int, seed: int) -> bytes:
    rng = random.Random(seed)
    b = bytearray(data)
    for _ in range(n):
        i = rng.randrange(len(b))
        b[i] = rng.choice(b"x,\n0.9 \x00\xff5")
    return bytes(b)


@pytest.mark.parametrize("qname", ["LR2S", "CM2S", "CM1S", "LR1S"])
def test_malformed_records_counted_and_dropped(qname):
    fam = qname[:2]
    params = g.LRParams(num_vehicles=100) if qname.startswith("LR1") else None
    data = stream(fam, "B(1)", 12, params=params)
    data = [_corrupt(d, 40, i) for i, d in enumerate(data)]
    if fam == "CM":
        data = [d if d.endswith(b"\n") else d + b"\n" for d in data]
        data[-1] = data[-1] + b"123,,456"            # unterminated tail record
        data[-1] = data[-1] + b"\n"                   # pushes must end with '\n' (host-side rule)
        data[3] = b"\n\n" + data[3]                   # empty lines
        data[5] = data[5] + (b"9" * 300 + b"\n")      # over-long line
    batches = split(data, [4, 4, 4])
    prod = product_run(qname, batches)
    compare_run(qname, prod, oracle_rows(qname, batches))
    assert any(rec["bad_records"] > 0 for _, rec, _ in prod)


def test_late_records():
    lr = lambda ts, spd: g.lr_format(dict(type=0, time=ts, vid=1, spd=spd, xway=0, lane=0, dir=0, seg=3,
                                          pos=0, qid=0, sinit=0, send=0, dow=0, tod=0, day=0))
    b1 = [b"".join(lr(t, 20) for t in (10, 11, 12, 13))]
    b2 = [b"".join(lr(t, 30) for t in (5, 12, 25, 13, 40))]     # 5 and 12 are late (W_prev = 13)
    b3 = [b"".join(lr(t, 10) for t in (41, 44, 39))]            # 39 late (W_prev = 40)
    batches = [b1, b2, b3]
    compare_run("LR2S", product_run("LR2S", batches, range_s=4, slide_s=2),
                oracle_rows("LR2S", batches, range_s=4, slide_s=2))


def test_custom_windows_and_negative_instances():
    data = stream("CM", "B(0.5)", 9)
    batches = split(data, [2, 3, 4])
    for R, S in ((4, 1), (6, 3), (5, 5), (1, 1)):
        compare_run("CM2S", product_run("CM2S", batches, range_s=R, slide_s=S),
                    oracle_rows("CM2S", batches, range_s=R, slide_s=S))


def test_device_and_host_segments_mixed():
    data = stream("CM", "B(1.1)", 20)
    batches = split(data, [5, 5, 10])
    devmask = [[i % 2 == 0 for i in range(len(b))] for b in batches]
    compare_run("CM2S", product_run("CM2S", batches, device_batches=devmask), oracle_rows("CM2S", batches))
    data = stream("LR", "B(1.3)", 20)
    batches = split(data, [5, 5, 10])
    devmask = [[i % 3 != 1 for i in range(len(b))] for b in batches]
    compare_run("LR2S", product_run("LR2S", batches, device_batches=devmask), oracle_rows("LR2S", batches))


def test_many_segments_more_than_one_launch():
    """> 128 borrowed device segments in one batch: several aggregate launches per batch, and
    segment cursors crossing many tiny segments inside one launch."""
    for fam, qname in (("LR", "LR2S"), ("CM", "CM2S"), ("LR", "LR1S")):
        # (LR1: every launch reads the retained-row FIFO's count when it starts and its last CTA
        # advances it; a segment's tail tile writes hole rows)
        params = g.LRParams(num_vehicles=150) if qname == "LR1S" else None
        data = stream(fam, "B(0.02)", 300, params=params)
        batches = [data[:170], data[170:190], data[190:]]
        devmask = [[True] * len(b) for b in batches]
        compare_run(qname, product_run(qname, batches, device_batches=devmask), oracle_rows(qname, batches))


def test_empty_flush_and_tiny_batches():
    compare_run("CM2S", product_run("CM2S", []), oracle_rows("CM2S", []))
    one = [[g.cm_record(g.SEED, 3, 0)]]
    compare_run("CM2S", product_run("CM2S", one), oracle_rows("CM2S", one))
    one = [[g.lr_record(g.SEED, 3, 0)]]
    compare_run("LR2S", product_run("LR2S", one), oracle_rows("LR2S", one))
    compare_run("LR1S", product_run("LR1S", one), oracle_rows("LR1S", one))
    compare_run("LR1S", product_run("LR1S", []), oracle_rows("LR1S", []))


def test_xways_domain_and_high_key_space():
    data = stream("LR", "B(2)", 31, params=g.LRParams(num_xways=16))
    batches = split(data, [10, 10, 11])
    compare_run("LR2S", product_run("LR2S", batches, num_xways=16), oracle_rows("LR2S", batches, num_xways=16))
    # with the default domain (10 xways) records with xway >= 10 are malformed
    compare_run("LR2S", product_run("LR2S", batches), oracle_rows("LR2S", batches))


def _cm_line(ts="7", miss="", job="1234567890", task="12", mach="345", ev="1", user="Ab+/Zz09",
             cat="2", prio="3", cpu="0.123456", ram="0.000001", disk="0.999999", cons="1"):
    return ",".join([ts, miss, job, task, mach, ev, user, cat, prio, cpu, ram, disk, cons]).encode() + b"\n"


def test_cm_field_shape_variants():
    """Every field-width variant of the CM grammar (reading R1) around the kernel's fast-path
    shapes (10-digit jobId, 8-char cpu/ram/disk, 1-char constraint): valid ones must be
    aggregated, invalid ones dropped — exactly as the oracle decides."""
    variants = [
        {}, {"job": "1"}, {"job": "123456789"}, {"job": "12345678901"}, {"job": "1234567890123456789"},
        {"job": "12345678901234567890"}, {"job": ""}, {"job": "12345x7890"}, {"ts": ""}, {"ts": "000000006"},
        {"ts": "0000000006"}, {"ts": "1a"}, {"miss": "x"}, {"task": ""}, {"task": "ab,c"}, {"task": "x y"},
        {"mach": ""}, {"mach": "12345678901234"}, {"ev": ""}, {"ev": "11"}, {"ev": "x"}, {"cat": ""},
        {"cat": "12"}, {"cat": "z"}, {"prio": ""}, {"prio": "123"}, {"cpu": "0.12345"}, {"cpu": "0.1234567"},
        {"cpu": "01234567"}, {"cpu": "0.12345x"}, {"ram": "1"}, {"ram": "0.1234567890"}, {"disk": ""},
        {"disk": "0.1"}, {"cons": ""}, {"cons": "10"}, {"cons": "xyz"}, {"user": ""}, {"user": "a" * 120},
        {"user": "a,b"}, {"ram": "0.12,3456"}, {"cons": "1,"},
    ]
    lines = []
    for i, v in enumerate(variants):
        for t in range(3):
            d = dict(ts=str(5 + t), job=f"{1000000000 + 7 * i}", ev="1")
            d.update(v)
            lines.append(_cm_line(**d))
    data = b"".join(lines)
    batches = [[data]]
    for q in ("CM2S", "CM1S"):
        prod = product_run(q, batches)
        compare_run(q, prod, oracle_rows(q, batches))


def test_cm_fast_path_fuzz():
    """Randomised lines around every boundary of the kernel's branch-free usual-shape decode
    (ts of 1..10 digits, line lengths 40..250 B, taskIndex/machineId widths, user lengths) plus
    single-byte mutations at and next to the separators the fast path reads off the masks:
    every line must be aggregated or dropped exactly as the oracle decides."""
    rng = random.Random(2111)
    digits = lambda n: "".join(rng.choice("0123456789") for _ in range(n))
    lines = []
    for i in range(6000):
        ts = str(5 + i * 8 // 6000).zfill(rng.randint(1, 10))     # widths 1..10, in-order seconds
        d = dict(ts=ts, job=digits(10) if rng.random() < 0.85 else digits(rng.randint(1, 20)),
                 task=digits(rng.randint(0, 5)), mach=digits(rng.randint(0, 11)),
                 ev=str(rng.choice([1, 1, 1, 0, 4, 5])) if rng.random() < 0.95 else digits(rng.randint(0, 2)),
                 user="".join(rng.choice("ABCdef+/019") for _ in range(rng.choice([0, 1, 5, 40, 70, 90, 150]))),
                 cat=str(rng.randrange(4)) if rng.random() < 0.95 else digits(rng.randint(0, 2)),
                 prio=digits(rng.randint(0, 3)),
                 cpu="0." + digits(6) if rng.random() < 0.9 else digits(rng.randint(0, 9)),
                 ram="0." + digits(6) if rng.random() < 0.9 else digits(rng.randint(0, 9)),
                 disk="0." + digits(6), cons=str(rng.randrange(2)) if rng.random() < 0.95 else digits(2))
        line = bytearray(_cm_line(**d))
        if rng.random() < 0.25:            # mutate a byte at / next to a separator
            seps = [k for k, c in enumerate(line) if c in b",."]
            k = min(max(rng.choice(seps) + rng.choice([-1, 0, 1]), 0), len(line) - 2)
            line[k] = rng.choice(b",.x05\n")
        lines.append(bytes(line))
    data = b"".join(lines)
    batches = [[data[:len(data) // 2].rsplit(b"\n", 1)[0] + b"\n"]]
    rest = data[len(batches[0][0]):]
    batches.append([rest])
    for q in ("CM2S", "CM1S"):
        prod = product_run(q, batches)
        compare_run(q, prod, oracle_rows(q, batches))


def test_cm_mixed_panes_in_warp_rounds():
    """Records whose timestamps jump around inside a batch (every warp round of 32 lines spans
    several panes) and categories 0..9: CM1's per-(pane, category) reduction takes its general
    path (the single-pane fast path only when a round is uniform), CM2's survivor drain mixes
    pane slots; both against the oracle.  Batch 2 overlaps batch 1's time range, so its records
    older than the watermark are dropped as late (reading R7) exactly as the oracle drops them."""
    rng = random.Random(4289)
    digits = lambda n: "".join(rng.choice("0123456789") for _ in range(n))

    def lines(t0, t1, n, uniform_every=0):
        out = []
        for i in range(n):
            # every `uniform_every`-th block of 64 lines keeps one ts (fast-path rounds in between)
            ts = t0 if uniform_every and (i // 64) % uniform_every == 0 else rng.randrange(t0, t1)
            out.append(_cm_line(ts=str(ts), job=str(10 ** 9 + rng.randrange(50)), ev=str(rng.choice([1, 1, 0, 4])),
                                cat=str(rng.randrange(10)), cpu="0." + digits(6),
                                user="".join(rng.choice("ABCdef+/019") for _ in range(rng.randint(20, 60)))))
        return b"".join(out)
    batches = [[lines(100, 160, 5000, uniform_every=3)], [lines(150, 230, 5000, uniform_every=2)]]
    for q in ("CM1S", "CM1T", "CM2S"):
        prod = product_run(q, batches)
        compare_run(q, prod, oracle_rows(q, batches))


def _pipelined_run(qname, batches, device_mask):
    """Push a batch's datasets, force it WITHOUT syncing (LMS_FLAG_PIPELINE: the previous batch
    may still run), sync only at the end; returns (rows of all batches, batch records)."""
    import torch
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import _lib as L
    keep = []
    with P.Query(qname, mode="manual", flags=L.LMS_FLAG_PIPELINE) as q:
        t = 0.0
        for bi, b in enumerate(batches):
            for di, d in enumerate(b):
                if device_mask[bi][di]:
                    buf = torch.empty(len(d) + 64, dtype=torch.uint8, device="cuda")
                    buf[:len(d)].copy_(torch.frombuffer(bytearray(d), dtype=torch.uint8))
                    torch.cuda.synchronize()
                    keep.append(buf)
                    q.push_device(buf.data_ptr(), len(d), t)
                else:
                    q.push(d, t)
                t += 1.0
            q.force(t)
        q.flush(t, ok=(L.LMS_OK, L.LMS_EFORMAT))
        rows = q.read_lr1() if qname.startswith("LR1") else q.read_agg()
        return rows, q.records()


@pytest.mark.parametrize("qname,traffic", [("CM2S", "B(1.3)"), ("LR2S", "U(0.6)"), ("CM1S", "B(0.9)"),
                                           ("LR1S", "B(0.4)")])
def test_pipelined_batches_equal_serial(qname, traffic):
    """LMS_FLAG_PIPELINE (up to three batches in flight, per-slot report / row buffers, staging-buffer
    guard for host pushes) gives the same rows and batch records as the serial path, which the
    other tests hold to the oracle."""
    import numpy as np
    fam = qname[:2]
    params = g.LRParams(num_vehicles=300) if qname == "LR1S" else None
    secs = stream(fam, traffic, 50, params=params)
    batches = split(secs, [3, 1, 5, 2, 4, 6, 1, 8])
    rng = random.Random(7)
    mask = [[rng.random() < 0.5 for _ in b] for b in batches]
    rows_p, recs_p = _pipelined_run(qname, batches, mask)
    serial = product_run(qname, batches, device_batches=mask)
    rows_s = np.concatenate([o[0] for o in serial])
    assert sorted(map(bytes, rows_p)) == sorted(map(bytes, rows_s))   # row order within a batch is free
    keys = ("num_records", "num_datasets", "batch_bytes", "windows_closed", "rows_emitted", "late_records",
            "bad_records", "watermark")
    assert [tuple(r[k] for k in keys) for r in recs_p] == [tuple(o[1][k] for k in keys) for o in serial]


def test_pipelined_three_deep_staging_and_deferred_status():
    """LMS_FLAG_PIPELINE with host pushes only (two staging buffers, up to three batches in
    flight): the pushes of batch i+2 refill the staging buffer batch i read, so they complete
    batch i first; a batch with malformed lines completed that way reports LMS_EFORMAT from a
    later call (deferred, never dropped).  Rows and batch records equal the serial run's."""
    import ctypes as C

    import numpy as np
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import _lib as L
    secs = stream("CM", "B(1.3)", 40, params=g.CMParams(num_jobs=200))
    batches = split(secs, [3, 2, 4, 1, 3, 5, 2, 3, 4])
    bad = b"abc,,1234567890,1,x,1,u,2,0,0.100000,0.1,0.1,0\n7,,bad\n"   # non-digit ts; 3 fields
    batches[1] = [batches[1][0] + bad] + batches[1][1:]
    serial = product_run("CM2S", batches)
    statuses = []
    with P.Query("CM2S", mode="manual", flags=L.LMS_FLAG_PIPELINE) as q:
        t = 0.0
        for b in batches:
            for d in b:
                arr = np.frombuffer(d, dtype=np.uint8)
                statuses.append(L.lms_push(q.h, C.c_void_p(arr.ctypes.data), len(d), t, None))
                t += 1.0
            statuses.append(L.lms_force_batch(q.h, t, None))
        statuses.append(L.lms_flush(q.h, t))
        rows_p = q.read_agg()
        recs_p = q.records()
    assert set(statuses) <= {L.LMS_OK, L.LMS_EFORMAT}
    assert statuses.count(L.LMS_EFORMAT) >= 1, "the malformed batch's status was dropped"
    assert sum(r["bad_records"] for r in recs_p) == 2
    rows_s = np.concatenate([o[0] for o in serial])
    assert sorted(map(bytes, rows_p)) == sorted(map(bytes, rows_s))
    keys = ("num_records", "num_datasets", "batch_bytes", "windows_closed", "rows_emitted", "late_records",
            "bad_records", "watermark")
    assert [tuple(r[k] for k in keys) for r in recs_p] == [tuple(o[1][k] for k in keys) for o in serial]


# ---------------------------------------------------------------- capacity limits (degenerate cases)

def _one_batch(qname, data, **cfg):
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import _lib as L
    with P.Query(qname, mode="manual", **cfg) as q:
        q.push(data, 0.0)
        q.force(1.0)
        st = q.sync(ok=(L.LMS_OK, L.LMS_EFORMAT, L.LMS_EOVERFLOW))
        st2 = q.flush(1.0, ok=(L.LMS_OK, L.LMS_EFORMAT, L.LMS_EOVERFLOW))
        rows = q.read_lr1() if qname.startswith("LR1") else q.read_agg()
        return st, st2, rows, q.records()


def test_key_capacity_overflow_is_reported_and_exact_for_admitted_keys():
    """CM2S with max_keys = 64 < 300 distinct jobIds: the batch reports LMS_EOVERFLOW and counts
    the dropped records; every key that did get a slot is aggregated exactly (its row equals the
    oracle's), none is half-counted."""
    from paper_2111_04289_b200 import _lib as L
    data = b"".join(stream("CM", "B(2)", 8, params=g.CMParams(num_jobs=300)))
    st, st2, rows, recs = _one_batch("CM2S", data, max_keys=64)
    assert L.LMS_EOVERFLOW in (st, st2)
    assert sum(r["overflow_records"] for r in recs) > 0
    ora = {(r.win_start, r.key[0]): r for o in oracle_rows("CM2S", [[data]]) for r in o.rows}
    assert len(rows) > 0
    for r in rows:
        o = ora[(int(r["win_start_s"]), int(r["key"]))]
        assert int(r["count"]) == o.count and int(r["sum_fixed"]) == o.sum_fixed


def test_pane_slot_exhaustion_is_reported():
    """pane_slots = 4 with records spread over 40 slides: panes that find no slot are dropped,
    counted, and the batch reports LMS_EOVERFLOW (never silently wrong)."""
    from paper_2111_04289_b200 import _lib as L
    data = b"".join(stream("LR", "B(0.2)", 200))
    st, st2, rows, recs = _one_batch("LR2S", data, pane_slots=4)
    assert L.LMS_EOVERFLOW in (st, st2)
    assert sum(r["overflow_records"] for r in recs) > 0


def test_result_row_capacity_overflow_is_reported():
    """max_result_rows smaller than one close's rows: LMS_EOVERFLOW, rows capped."""
    from paper_2111_04289_b200 import _lib as L
    data = b"".join(stream("CM", "B(2)", 70, params=g.CMParams(num_jobs=500)))
    st, st2, rows, recs = _one_batch("CM2S", data, max_result_rows=100)
    assert L.LMS_EOVERFLOW in (st, st2)
    assert len(rows) <= 200


def test_batch_buffer_capacity_on_push():
    """A push beyond max_batch_bytes is refused with LMS_EOVERFLOW (nothing is truncated)."""
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import _lib as L
    data = b"".join(stream("LR", "B(1)", 3))
    with P.Query("LR2S", mode="manual", max_batch_bytes=len(data) - 70) as q:
        with pytest.raises(P.LmsError) as ei:
            q.push(data, 0.0)
        assert ei.value.status == L.LMS_EOVERFLOW
        q.push(data[:70 * 100], 0.0)          # a smaller push still fits
        q.force(1.0)
        q.sync()
        assert q.record(0)["num_records"] == 100


@pytest.mark.parametrize("qname,traffic", [("LR1S", "B(0.4)"), ("LR1T", "B(0.3)")])
def test_lr1_dense_vehicles_match_oracle(qname, traffic):
    """LMS_FLAG_DENSE_VEHICLES (vehicle ids index the counts, no dictionary): same rows as the
    oracle for VIDs < max_keys (the generator's V = 10^6 < 2^20)."""
    from paper_2111_04289_b200 import _lib as L
    secs = stream("LR", traffic, 65, params=g.LRParams(num_vehicles=400))
    batches = split(secs, [7, 11, 3, 30])
    compare_run(qname, product_run(qname, batches, flags=L.LMS_FLAG_DENSE_VEHICLES),
                oracle_rows(qname, batches))


@pytest.mark.parametrize("sel_ppm,jobs,max_keys", [(1_000_000, 2_000, 1 << 16), (10_000, 2_000, 1 << 16),
                                                   (260_000, 200_000, 1 << 18)])
def test_cm2_selectivity_and_key_space_sweep(sel_ppm, jobs, max_keys):
    """CM2 across the §8(d) sweeps: eventType==1 selectivity 1.0 and 0.01 (every / almost no
    record survives the WHERE), and a large jobId key space (2*10^5 distinct keys in the
    dictionary, max_keys 2^18) — exact against the oracle."""
    secs = stream("CM", "B(4)", 14, params=g.CMParams(num_jobs=jobs, sel_ppm=sel_ppm))
    batches = split(secs, [5, 4, 5])
    compare_run("CM2S", product_run("CM2S", batches, max_keys=max_keys), oracle_rows("CM2S", batches))
