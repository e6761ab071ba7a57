"""Pins for the input generator (lmsgen) that oracle and CUDA path share.

Closed forms and invariants fixed by the paper's traffic definitions
and by the record sizes; SplitMix64 published test vectors;
golden digests written by tests/golden/make_gen_golden.py (calls lmsgen only).
"""
import hashlib
import json
import os

import pytest

import lmsgen as g
from oracle import records as R

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_splitmix64_reference_vectors():
    # SplitMix64 seeded with 0: first output 0xE220A8397B1DCDAF (Vigna's reference);
    # seeded with 1234567: the first five outputs of the reference implementation.
    assert g.mix(0) == 0xE220A8397B1DCDAF
    s, out = 1234567, []
    for _ in range(5):
        out.append(g.mix(s))
        s = (s + 0x9E3779B97F4A7C15) & g.M64
    assert out == [6457827717110365317, 3203168211198807973, 9817491932198370423,
                   4593380528125082431, 16408922859458223821]


def test_u_range_and_extremes():
    assert g.u(0, 10) == 0
    assert g.u(g.M64, 10) == 9
    assert all(0 <= g.u(g.mix(i), 7) < 7 for i in range(1000))


def test_basic_traffic_closed_form():
    # B(N): "a constant number of (N*1000) records every second"
    for n, rate in (("1", 1000), ("100", 100000), ("10000", 10 ** 7), ("2.5", 2500)):
        tr = g.Traffic.parse(f"B({n})")
        assert [tr.count(t) for t in range(5)] == [rate] * 5


def test_range_traffic_bounds_and_mean():
    # R(L,U): "lower limit value (L*1000) and an upper limit value (U*1000)"
    tr = g.Traffic.parse("R(50,500)")
    cs = [tr.count(t) for t in range(4000)]
    assert min(cs) >= 50000 and max(cs) <= 500000
    assert abs(sum(cs) / len(cs) - 275000) < 0.03 * 275000
    tr = g.Traffic.parse("R(0.1,5)")
    cs = [tr.count(t) for t in range(2000)]
    assert min(cs) >= 100 and max(cs) <= 5000


def test_uniform_traffic_converges_to_mean():
    # U(N): "converges to a specific average value (N*1000)"; +-2% over 1e4 s
    tr = g.Traffic.parse("U(1)")
    cs = [tr.count(t) for t in range(10000)]
    mean = sum(cs) / len(cs)
    assert abs(mean - 1000) < 20
    var = sum((c - mean) ** 2 for c in cs) / len(cs)
    assert 0.8 * 250 ** 2 < var < 1.2 * 250 ** 2          # sigma = mean/4
    assert min(cs) >= 1


def test_traffic_parse_rejects_garbage():
    for bad in ("X(1)", "B()", "R(5)", "B(0)", "R(5,1)", "B(0.0001)"):
        with pytest.raises(ValueError):
            g.Traffic.parse(bad)


def test_lr_records_fixed_70_bytes_and_roundtrip():
    for t in (0, 7, 123456):
        for i in range(200):
            f = g.lr_fields(g.SEED, t, i)
            b = g.lr_format(f)
            assert len(b) == 70                                   # P:22 "70 B (per record, fixed)"
            r = R.parse_lr_record(b)
            assert r is not None
            assert (r.ts, r.vehicle, r.speed, r.xway, r.lane, r.dir, r.seg) == \
                (f["time"], f["vid"], f["spd"], f["xway"], f["lane"], f["dir"], f["seg"])
            assert 0 <= f["spd"] <= 100 and f["xway"] < 10 and f["seg"] < 100


def test_cm_records_130_145_bytes_and_roundtrip():
    lens = set()
    for t in (0, 59, 99999):
        for i in range(300):
            f = g.cm_fields(g.SEED, t, i)
            b = g.cm_format(g.SEED, t, i, f)
            assert 130 <= len(b) <= 145                            # P:28 "130 ~ 145 B"
            lens.add(len(b))
            assert b.endswith(b"\n") and b.count(b"\n") == 1
            r = R.parse_cm_record(b[:-1])
            assert r is not None
            assert (r.ts, r.job, r.event, r.cat, r.cpu_m) == \
                (f["ts"], f["job"], f["event"], f["cat"], f["cpu_m"])
    assert lens == set(range(130, 146))


def test_cm_event_mix_selectivity():
    ev = [g.cm_fields(g.SEED, 3, i)["event"] for i in range(20000)]
    sel = ev.count(1) / len(ev)
    assert abs(sel - 0.26) < 0.015
    p = g.CMParams(sel_ppm=100000)
    ev = [g.cm_fields(g.SEED, 3, i, p)["event"] for i in range(20000)]
    assert abs(ev.count(1) / len(ev) - 0.10) < 0.01


def test_cm_job_cardinality():
    p = g.CMParams(num_jobs=50)
    jobs = {g.cm_fields(g.SEED, 1, i, p)["job"] for i in range(3000)}
    assert len(jobs) == 50
    assert all(10 ** 9 <= j < 10 ** 10 for j in jobs)


def test_lr_speed_structure_having_fraction():
    # per-key congestion means mu_k ~ U{10..90}: about 35% of keys have mean < 40
    mus = [g._mu(g.SEED, k) for k in range(2000)]
    assert min(mus) >= 10 and max(mus) <= 90
    frac = sum(1 for m in mus if m < 40) / len(mus)
    assert 0.3 < frac < 0.42


def test_determinism():
    a = g.second_bytes("CM", 5, 100)
    b = g.second_bytes("CM", 5, 100)
    assert a == b
    assert g.second_bytes("CM", 5, 100, seed=1) != a


def test_golden_digests():
    with open(os.path.join(GOLDEN, "gen_digests.json")) as fh:
        gold = json.load(fh)
    for key, want in gold["digests"].items():
        fam, traffic = key.split(":")
        h = hashlib.sha256()
        for t, data in g.stream_datasets(fam, traffic, 3):
            h.update(data)
        assert h.hexdigest() == want, key


def test_vectorised_columns_match_scalar_generator():
    """lmsgen.vec (numpy column form, used by the full-size checks) == lmsgen.lr_fields /
    cm_fields record by record, incl. the u() high-product at large n (jobId map)."""
    import numpy as np
    from lmsgen import vec
    rng = np.random.default_rng(5)
    assert [int(v) for v in vec.mix(np.array([0, 1, 2 ** 64 - 1], dtype=np.uint64))] == \
        [g.mix(0), g.mix(1), g.mix(2 ** 64 - 1)]
    xs = rng.integers(0, 2 ** 63, 1000, dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    for n in (2, 100, 500000, 9 * 10 ** 9, 2 ** 63 + 12345):
        assert [int(v) for v in vec.u(xs, n)] == [g.u(int(x), n) for x in xs]
    for t, p in ((0, g.LRParams()), (17, g.LRParams(num_xways=3, num_vehicles=77))):
        cols = vec.lr_columns(g.SEED, t, 3000, p)
        for i in rng.integers(0, 3000, 200):
            f = g.lr_fields(g.SEED, t, int(i), p)
            assert (f["vid"], f["xway"], f["dir"], f["seg"], f["lane"], f["spd"]) == tuple(
                int(cols[k][i]) for k in ("vid", "xway", "dir", "seg", "lane", "spd"))
    for t, p in ((0, g.CMParams()), (5, g.CMParams(num_jobs=300, sel_ppm=700000))):
        cols = vec.cm_columns(g.SEED, t, 3000, p)
        for i in rng.integers(0, 3000, 200):
            f = g.cm_fields(g.SEED, t, int(i), p)
            assert (f["job"], f["event"], f["cat"], f["cpu_m"]) == tuple(
                int(cols[k][i]) for k in ("job", "event", "cat", "cpu_m"))
