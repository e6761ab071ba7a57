"""Pins for oracle/queries.py: Table IV semantics on windows.

Pins used (none re-types the oracle's own code):
  * hand-computed expected rows on tiny streams (written out below);
  * sqlite3 (a library SQL engine) running the Table IV SQL per instance;
  * exact rational sums (fractions) for the fp64 SUM/AVG;
  * invariants: every record lies in R/S instances; tumbling == GROUP BY ts // R;
    batching invariance of the emitted result; LR1 output cardinality.
"""
import random
import sqlite3
from fractions import Fraction

import pytest

import lmsgen as g
from oracle import queries as Q
from oracle import records as R


def lr(ts, xway=0, d=0, seg=0, spd=0, vid=0, lane=0):
    return g.lr_format(dict(type=0, time=ts, vid=vid, spd=spd, xway=xway, lane=lane, dir=d, seg=seg,
                            pos=0, qid=0, sinit=0, send=0, dow=0, tod=0, day=0))


def cm(ts, job=1000000000, ev=1, cat=0, cpu="0.000001"):
    return f"{ts},,{job},0,0,{ev},u,{cat},0,{cpu},0,0,0\n".encode()


# ----------------------------------------------------------------- hand-computed examples

LR2_TINY = [lr(0, 0, 0, 1, 30), lr(1, 0, 0, 1, 50), lr(2, 0, 0, 1, 20), lr(3, 1, 1, 5, 45),
            lr(4, 0, 0, 1, 10), lr(5, 1, 1, 5, 35), lr(6, 0, 0, 1, 60), lr(7, 1, 1, 5, 39)]
# windows [2k, 2k+4), HAVING avg < 40.0, computed by hand:
#  k=-1 [-2,2): (0,0,1) 80/2 = 40.0 -> dropped by HAVING
#  k= 0 [0,4):  (0,0,1) 100/3; (1,1,5) 45 -> dropped
#  k= 1 [2,6):  (0,0,1) 30/2;  (1,1,5) 80/2 = 40 -> dropped
#  k= 2 [4,8):  (0,0,1) 70/2;  (1,1,5) 74/2
#  k= 3 [6,10): (0,0,1) 60 -> dropped; (1,1,5) 39
LR2_TINY_EXPECTED = {(0, (0, 0, 1), 100, 3), (2, (0, 0, 1), 30, 2), (4, (0, 0, 1), 70, 2),
                     (4, (1, 1, 5), 74, 2), (6, (1, 1, 5), 39, 1)}


def test_lr2_tiny_by_hand():
    q = Q.query_spec("LR2S", range_s=4, slide_s=2)
    recs, bad = R.parse_dataset("LR", b"".join(LR2_TINY))
    assert bad == 0
    got = {(r.win_start, r.key, r.sum_fixed, r.count)
           for rows in Q.brute_force_all(q, recs).values() for r in rows}
    assert got == LR2_TINY_EXPECTED
    for rows in Q.brute_force_all(q, recs).values():
        for r in rows:
            assert r.avg == Fraction(r.sum_fixed, r.count).__float__()
            assert r.win_end == r.win_start + 4


def test_lr2_tiny_emission_by_hand():
    q = Q.query_spec("LR2S", range_s=4, slide_s=2)
    b1, b2, b3 = [b"".join(LR2_TINY[0:3])], [b"".join(LR2_TINY[3:6])], [b"".join(LR2_TINY[6:8])]
    outs = Q.replay(q, [b1, b2, b3])
    rows = [{(r.win_start, r.key, r.sum_fixed, r.count) for r in o.rows} for o in outs]
    # W = 2 -> emit k <= -1 (no rows); W = 5 -> k = 0; W = 7 -> k = 1; flush -> k = 2, 3
    assert [o.watermark for o in outs] == [2, 5, 7, 7]
    assert [o.windows_closed for o in outs] == [1, 1, 1, 2]
    assert rows[0] == set()
    assert rows[1] == {(0, (0, 0, 1), 100, 3)}
    assert rows[2] == {(2, (0, 0, 1), 30, 2)}
    assert rows[3] == {(4, (0, 0, 1), 70, 2), (4, (1, 1, 5), 74, 2), (6, (1, 1, 5), 39, 1)}


def test_cm2_tiny_by_hand():
    q = Q.query_spec("CM2S", range_s=2, slide_s=1)
    data = (cm(0, 11, 1, cpu="0.250000") + cm(0, 11, 0, cpu="0.900000") + cm(1, 11, 1, cpu="0.500000")
            + cm(1, 22, 1, cpu="0.125000") + cm(2, 22, 1, cpu="1.000000"))
    recs, _ = R.parse_dataset("CM", data)
    got = {(r.win_start, r.key, r.count, r.sum_fixed, r.sum, r.avg)
           for rows in Q.brute_force_all(q, recs).values() for r in rows}
    # instances [k, k+2); eventType==1 only (the 0.9 record is filtered out)
    assert got == {(-1, (11,), 1, 250000, 0.25, 0.25),
                   (0, (11,), 2, 750000, 0.75, 0.375), (0, (22,), 1, 125000, 0.125, 0.125),
                   (1, (11,), 1, 500000, 0.5, 0.5), (1, (22,), 2, 1125000, 1.125, 0.5625),
                   (2, (22,), 1, 1000000, 1.0, 1.0)}


def test_cm1_tiny_order_by_sum():
    q = Q.query_spec("CM1T", range_s=10)
    data = (cm(0, cat=3, cpu="0.500000") + cm(1, cat=1, cpu="0.100000") + cm(2, cat=2, cpu="0.300000")
            + cm(3, cat=1, cpu="0.100000") + cm(4, cat=0, cpu="0.200000", ev=4))
    recs, _ = R.parse_dataset("CM", data)
    rows = Q.brute_force_all(q, recs)[0]
    # sums: cat1 0.2 (tie with cat0 0.2 -> category order), cat2 0.3, cat3 0.5
    assert [(r.key[0], r.rank) for r in sorted(rows, key=lambda r: r.rank)] == [(0, 0), (1, 1), (2, 2), (3, 3)]
    assert {r.key[0]: r.sum_fixed for r in rows} == {0: 200000, 1: 200000, 2: 300000, 3: 500000}


def test_lr1_tiny_multiplicity_by_hand():
    q = Q.query_spec("LR1S", range_s=4, slide_s=2)
    data = lr(0, vid=7) + lr(1, vid=8) + lr(2, vid=7) + lr(3, vid=7) + lr(3, vid=9)
    recs, _ = R.parse_dataset("LR", data)
    got = sorted((r.win_start, r.ts, r.vehicle, r.m)
                 for rows in Q.brute_force_all(q, recs).values() for r in rows)
    # k=-1: L = newest slide [0,2) = {ts0 v7, ts1 v8}, A = same -> m = 1, 1
    # k=0:  L = [2,4) = {ts2 v7, ts3 v7, ts3 v9}; A = all five -> m = 3, 3, 1
    # k=1:  L = [4,6) empty
    assert got == [(-2, 0, 7, 1), (-2, 1, 8, 1), (0, 2, 7, 3), (0, 3, 7, 3), (0, 3, 9, 1)]


def test_lr1_tumbling_l_equals_a():
    q = Q.query_spec("LR1T", range_s=4)
    data = lr(0, vid=7) + lr(1, vid=8) + lr(2, vid=7) + lr(5, vid=7)
    recs, _ = R.parse_dataset("LR", data)
    got = sorted((r.win_start, r.ts, r.vehicle, r.m)
                 for rows in Q.brute_force_all(q, recs).values() for r in rows)
    assert got == [(0, 0, 7, 2), (0, 1, 8, 1), (0, 2, 7, 2), (4, 5, 7, 1)]


def test_instances_of_closed_form():
    q = Q.query_spec("CM2S")     # R=60, S=5
    for ts in (0, 1, 59, 60, 61, 12345):
        ks = list(Q.instances_of(ts, q))
        assert len(ks) == 12
        assert all(k * 5 <= ts < k * 5 + 60 for k in ks)
        assert not (ks[0] - 1) * 5 + 60 > ts and not (ks[-1] + 1) * 5 <= ts


# ----------------------------------------------------------------- sqlite3 cross-check

def _random_stream(family, seconds, rate, seed=3, params=None):
    return b"".join(d for _, d in g.stream_datasets(family, f"B({rate / 1000})", seconds, seed=seed,
                                                     params=params))


def _sqlite_lr(recs):
    con = sqlite3.connect(":memory:")
    con.execute("CREATE TABLE SegSpeedStr (id INTEGER, timestamp INTEGER, vehicle INTEGER, speed INTEGER,"
                " highway INTEGER, lane INTEGER, direction INTEGER, segment INTEGER)")
    con.executemany("INSERT INTO SegSpeedStr VALUES (?,?,?,?,?,?,?,?)",
                    [(i, x.ts, x.vehicle, x.speed, x.xway, x.lane, x.dir, x.seg) for i, x in enumerate(recs)])
    return con


def test_lr2_matches_sqlite_table_iv_sql():
    q = Q.query_spec("LR2S")
    recs, _ = R.parse_dataset("LR", _random_stream("LR", 70, 40, params=g.LRParams(num_xways=1)))
    con = _sqlite_lr(recs)
    got = Q.brute_force_all(q, recs)
    for k, rows in got.items():
        s = k * q.slide_s
        sql = ("SELECT highway, direction, segment, SUM(speed), COUNT(*), AVG(speed) as avgSpeed "
               "FROM SegSpeedStr WHERE timestamp >= ? AND timestamp < ? "
               "GROUP BY highway, direction, segment HAVING (avgSpeed < 40.0)")
        want = {(h, d, sg): (sm, c, a) for h, d, sg, sm, c, a in con.execute(sql, (s, s + q.range_s))}
        have = {r.key: (r.sum_fixed, r.count, r.avg) for r in rows}
        assert have == want, k


def test_lr1_matches_sqlite_self_join():
    q = Q.query_spec("LR1S")
    recs, _ = R.parse_dataset("LR", _random_stream("LR", 40, 25, params=g.LRParams(num_vehicles=30)))
    con = _sqlite_lr(recs)
    got = Q.brute_force_all(q, recs)
    for k, rows in got.items():
        s = k * q.slide_s
        e = s + q.range_s
        sql = ("SELECT L.timestamp, L.vehicle, L.speed, L.highway, L.lane, L.direction, L.segment, COUNT(*) "
               "FROM SegSpeedStr AS A, SegSpeedStr AS L "
               "WHERE A.vehicle == L.vehicle AND A.timestamp >= ? AND A.timestamp < ? "
               "AND L.timestamp >= ? AND L.timestamp < ? GROUP BY L.id")
        want = sorted(con.execute(sql, (s, e, e - q.slide_s, e)))
        have = sorted((r.ts, r.vehicle, r.speed, r.xway, r.lane, r.dir, r.seg, r.m) for r in rows)
        assert have == want, k


def _sqlite_cm(recs):
    con = sqlite3.connect(":memory:")
    con.execute("CREATE TABLE TaskEvents (timestamp INTEGER, jobId INTEGER, eventType INTEGER, "
                "category INTEGER, cpu REAL, cpu_m INTEGER)")
    con.executemany("INSERT INTO TaskEvents VALUES (?,?,?,?,?,?)",
                    [(x.ts, x.job, x.event, x.cat, x.cpu, x.cpu_m) for x in recs])
    return con


def test_cm1_cm2_match_sqlite_table_iv_sql():
    recs, _ = R.parse_dataset("CM", _random_stream("CM", 75, 30, params=g.CMParams(num_jobs=20)))
    con = _sqlite_cm(recs)
    q = Q.query_spec("CM1S")
    for k, rows in Q.brute_force_all(q, recs).items():
        s = k * q.slide_s
        sql = ("SELECT category, SUM(cpu) as totalCpu, SUM(cpu_m), COUNT(*) FROM TaskEvents "
               "WHERE timestamp >= ? AND timestamp < ? GROUP BY category ORDER BY SUM(cpu), category")
        want = list(con.execute(sql, (s, s + q.range_s)))
        have = sorted(rows, key=lambda r: r.rank)
        assert [(r.key[0], r.sum_fixed, r.count) for r in have] == [(c, m, n) for c, _, m, n in want]
        for r, (_, tot, _, _) in zip(have, want):
            assert r.sum == pytest.approx(tot, rel=1e-12)
    q = Q.query_spec("CM2S")
    for k, rows in Q.brute_force_all(q, recs).items():
        s = k * q.slide_s
        sql = ("SELECT jobId, AVG(cpu) as avgCpu, SUM(cpu_m), COUNT(*) FROM TaskEvents "
               "WHERE timestamp >= ? AND timestamp < ? AND (eventType == 1) GROUP BY jobId")
        want = {j: (a, m, n) for j, a, m, n in con.execute(sql, (s, s + q.range_s))}
        have = {r.key[0]: (r.avg, r.sum_fixed, r.count) for r in rows}
        assert set(have) == set(want)
        for j in want:
            assert have[j][1:] == want[j][1:]
            assert have[j][0] == pytest.approx(want[j][0], rel=1e-12)


# ----------------------------------------------------------------- exact sums, invariants

def test_cm_fp64_sums_within_budget_of_exact_rational():
    recs, _ = R.parse_dataset("CM", _random_stream("CM", 12, 800, params=g.CMParams(num_jobs=3)))
    for qn in ("CM1S", "CM2S"):
        q = Q.query_spec(qn)
        for rows in Q.brute_force_all(q, recs).values():
            for r in rows:
                exact = Fraction(r.sum_fixed, 10 ** 6)
                assert abs(Fraction(r.sum) - exact) <= Fraction(1, 10 ** 9) * exact
                assert abs(Fraction(r.avg) - exact / r.count) <= Fraction(1, 10 ** 9) * exact / r.count


def test_every_record_in_r_over_s_instances():
    recs, _ = R.parse_dataset("CM", _random_stream("CM", 30, 20))
    for qn in ("CM1S", "CM1T"):
        q = Q.query_spec(qn)
        total = sum(r.count for rows in Q.brute_force_all(q, recs).values() for r in rows)
        assert total == len(recs) * (q.range_s // q.slide_s)


def test_tumbling_equals_textbook_group_by():
    recs, _ = R.parse_dataset("CM", _random_stream("CM", 130, 10))
    q = Q.query_spec("CM1T")
    by = {}
    for x in recs:
        by.setdefault((x.ts // 60, x.cat), []).append(x.cpu_m)
    have = {(r.win_start // 60, r.key[0]): (r.count, r.sum_fixed)
            for rows in Q.brute_force_all(q, recs).values() for r in rows}
    assert have == {k: (len(v), sum(v)) for k, v in by.items()}


def test_lr1_output_cardinality_and_m_at_least_one():
    recs, _ = R.parse_dataset("LR", _random_stream("LR", 33, 20, params=g.LRParams(num_vehicles=40)))
    q = Q.query_spec("LR1S")
    rows = [r for rows in Q.brute_force_all(q, recs).values() for r in rows]
    assert len(rows) == len(recs)          # every record is in exactly one newest slide
    assert all(r.m >= 1 for r in rows)


@pytest.mark.parametrize("qn", ["LR2S", "CM2S", "CM1S", "LR1S", "CM1T"])
def test_batching_invariance(qn):
    q = Q.query_spec(qn)
    fam = q.family
    params = g.LRParams(num_vehicles=50) if fam == "LR" else g.CMParams(num_jobs=30)
    secs = [d for _, d in g.stream_datasets(fam, "B(0.015)", 75, seed=9, params=params)]
    recs, _ = R.parse_dataset(fam, b"".join(secs))
    want = sorted(map(repr, (r for rows in Q.brute_force_all(q, recs).values() for r in rows)))
    rng = random.Random(qn)
    for _ in range(3):
        batches, cur = [], []
        for d in secs:
            cur.append(d)
            if rng.random() < 0.3:
                batches.append(cur)
                cur = []
        if cur:
            batches.append(cur)
        outs = Q.replay(q, batches)
        got = sorted(map(repr, (r for o in outs for r in o.rows)))
        assert got == want
        assert sum(o.late for o in outs) == 0


def test_late_records_dropped_and_counted():
    q = Q.query_spec("LR2S", range_s=4, slide_s=2)
    b1 = [lr(10, spd=10) + lr(12, spd=10)]
    b2 = [lr(11, spd=10) + lr(12, spd=20) + lr(13, spd=30)]   # ts 11 < W_prev = 12 -> late
    outs = Q.replay(q, [b1, b2])
    assert outs[1].late == 1 and outs[0].late == 0
    allrows = {(r.win_start, r.count, r.sum_fixed) for o in outs for r in o.rows}
    # [10,14) keeps ts 10, 12, 12, 13 (the late ts 11 is dropped): 4 rows, sum 70
    assert (10, 4, 70) in allrows and (12, 3, 60) in allrows
