"""Pins for oracle/sizer.py, planner.py, regression.py, metrics.py.

SPEC.md worked examples and the
properties it states, plus Eq. 4/5 identities.
"""
import itertools
import math
import random

import pytest

from oracle import metrics as M
from oracle import planner as P
from oracle import regression as G
from oracle import sizer as Z

MB = 1e6


def ds(i, t, nbytes):
    return Z.Dataset(i, t, nbytes)


# ------------------------------------------------------------------ Eq. 6 / Algorithm 1

def test_eq6_examples():
    # S:202  maxBuff 2 s, total 4 MB, AvgThPut 2 MB/s -> 4.0 s
    assert Z.est_max_lat(10.0, [ds(0, 8.0, 2 * MB), ds(1, 9.0, 2 * MB)], 2 * MB) == pytest.approx(4.0)
    # S:203  single dataset ingested at now, 1 MB at 1 MB/s -> 1.0 s
    assert Z.est_max_lat(5.0, [ds(0, 5.0, MB)], MB) == pytest.approx(1.0)
    with pytest.raises(ValueError):
        Z.est_max_lat(1.0, [], MB)
    with pytest.raises(ValueError):
        Z.est_max_lat(1.0, [ds(0, 0, 1)], 0.0)


def test_alg1_examples():
    # S:192 nothing buffered, nothing new -> keep polling
    d = Z.construct_micro_batch([], [], 1.0, mode="lmstream", slide_s=3, deadline_s=0,
                                avg_thput_prev=MB, max_lat_history=[])
    assert not d.admitted and d.batch == [] and d.carried == []
    # S:193 slide 3 s; max Buff 2.5 s; 1.2 MB at 2 MB/s -> EstMaxLat 3.1 >= 3 -> admit
    d = Z.construct_micro_batch([ds(0, 7.5, 0.7 * MB)], [ds(1, 9.0, 0.5 * MB)], 10.0, mode="lmstream",
                                slide_s=3, deadline_s=0, avg_thput_prev=2 * MB, max_lat_history=[1.0])
    assert d.admitted and d.est_max_lat == pytest.approx(3.1) and [x.id for x in d.batch] == [0, 1]
    # S:194 tumbling; mean past MaxLat 4 s; EstMaxLat 2.0 -> cancel, carried = tmp
    d = Z.construct_micro_batch([ds(0, 9.0, MB)], [ds(1, 10.0, 0)], 10.0, mode="lmstream", slide_s=0,
                                deadline_s=0, avg_thput_prev=MB, max_lat_history=[3.0, 5.0])
    assert not d.admitted and d.est_max_lat == pytest.approx(2.0) and [x.id for x in d.carried] == [0, 1]


def test_alg1_bootstrap_tumbling_and_cap():
    d = Z.construct_micro_batch([], [ds(0, 0, 10)], 0.0, mode="lmstream", slide_s=5, deadline_s=0,
                                avg_thput_prev=None, max_lat_history=[])
    assert d.admitted and d.reason == "bootstrap"
    d = Z.construct_micro_batch([], [ds(0, 0, 10)], 0.0, mode="lmstream", slide_s=0, deadline_s=0,
                                avg_thput_prev=MB, max_lat_history=[9.0])
    assert d.admitted                                                  # < 2 completed
    many = [ds(i, 0.0, 1) for i in range(4096)]
    d = Z.construct_micro_batch(many, [], 0.0, mode="lmstream", slide_s=100, deadline_s=0,
                                avg_thput_prev=1e12, max_lat_history=[])
    assert d.admitted and d.reason == "cap"


def test_alg1_sorts_new_files_by_creation_time():
    d = Z.construct_micro_batch([ds(5, 1.0, 1)], [ds(9, 3.0, 1), ds(7, 2.0, 1)], 100.0, mode="lmstream",
                                slide_s=1, deadline_s=0, avg_thput_prev=1.0, max_lat_history=[])
    assert [x.id for x in d.batch] == [5, 7, 9]


def test_deadline_modes():
    # CG(dN), N > 0: sliding branch with SlideTime := N (reading R16)
    args = dict(buffered=[ds(0, 0.0, MB)], new_files=[], now=0.5, slide_s=30, avg_thput_prev=MB,
                max_lat_history=[1, 1, 1])
    assert Z.construct_micro_batch(mode="deadline", deadline_s=1.5, **args).admitted
    assert not Z.construct_micro_batch(mode="deadline", deadline_s=1.6, **args).admitted
    # CG(d0): tumbling branch (mean of past MaxLat = 1)
    assert Z.construct_micro_batch(mode="deadline", deadline_s=0, **args).admitted


def _run_virtual(adm, arrivals, proc_fn, horizon, poll=0.01):
    """Virtual clock: arrivals [(t, bytes)], proc_fn(batch_bytes) -> seconds."""
    t, i, busy_until, log, nid = 0.0, 0, None, [], 0
    while t < horizon:
        while i < len(arrivals) and arrivals[i][0] <= t + 1e-12:
            adm.push(ds(nid, arrivals[i][0], arrivals[i][1]))
            nid += 1
            i += 1
        if busy_until is not None and t >= busy_until - 1e-12:
            log.append(adm.complete(proc))
            busy_until = None
        if busy_until is None:
            d = adm.poll(t)
            if d.admitted:
                proc = proc_fn(sum(x.nbytes for x in d.batch))
                busy_until = t + proc
        t = round(t + poll, 6)
    return log


def test_lmstream_bounds_latency_near_slide_while_trigger_grows():
    arrivals = [(float(s), 1000) for s in range(400)]
    proc = lambda b: 0.5 + b / 1500.0                 # capacity 1500 B/s > 1000 B/s arrival rate
    lm = _run_virtual(Z.Admission("lmstream", slide_s=3.0), arrivals, proc, 400)
    assert lm and max(lm[5:]) < 3.0 + 1.5             # bounded near the slide time (Eq. 2)
    heavy = lambda b: 6.0 * b / 5000.0                # Fig. 5: proc_0 = 6 s for a 5-dataset batch, 5 s trigger
    os_ = _run_virtual(Z.Admission("trigger", trigger_s=5.0), arrivals, heavy, 400)
    assert all(b > a for a, b in zip(os_[2:], os_[3:]))   # static trigger: latency keeps increasing


def test_cancel_never_drops_data_and_first_crossing():
    rng = random.Random(4)
    adm = Z.Admission("lmstream", slide_s=2.0)
    seen, t, pushed, admitted_ids = [], 0.0, 0, []
    last_est = None
    for step in range(3000):
        if rng.random() < 0.05:
            adm.push(ds(pushed, t, rng.randrange(1, 5000)))
            pushed += 1
        d = adm.poll(t)
        if d.admitted:
            admitted_ids += [x.id for x in d.batch]
            if d.est_max_lat is not None and last_est is not None:
                assert last_est < 2.0                       # previous poll was below target
            adm.complete(0.05)
            last_est = None
        elif d.reason == "buffer":
            assert sorted(x.id for x in d.carried) == sorted(x.id for x in adm.buffered)
            last_est = d.est_max_lat
        t = round(t + 0.01, 6)
    rest = [x.id for x in adm.force(t).batch]
    assert sorted(admitted_ids + rest) == list(range(pushed))


def test_eq4_eq5_identities():
    adm = Z.Admission("manual")
    for k in range(5):
        adm.push(ds(k, float(k), 100 * (k + 1)))
        d = adm.force(float(k) + 0.5)
        ml = adm.complete(0.25 * (k + 1))
        assert ml == pytest.approx(0.5 + 0.25 * (k + 1))              # Eq. 5
    assert adm.avg_thput == pytest.approx(sum(100 * (k + 1) for k in range(5)) /
                                          sum(0.25 * (k + 1) for k in range(5)))   # Eq. 4


# ------------------------------------------------------------------ Eq. 7-9, Algorithm 2

def test_eq7_8_9_examples():
    assert P.cpu_cost(1.0, 15e3, 150e3) == pytest.approx(0.1)
    assert P.cpu_cost(0.8, 1500e3, 150e3) == pytest.approx(8.0)
    assert P.cpu_cost(0.9, 150e3, 150e3) == pytest.approx(0.9)
    assert P.gpu_cost(1.0, 15e3, 150e3) == pytest.approx(10.0)
    assert P.gpu_cost(0.8, 1500e3, 150e3) == pytest.approx(0.08)
    assert P.trans_cost(0.1, 150e3, 150e3) == pytest.approx(0.1)
    assert P.trans_cost(0.1, 15e3, 150e3) == pytest.approx(0.01)
    assert P.trans_cost(0.1, 1.5e6, 150e3) == pytest.approx(1.0)
    for base in (0.8, 0.9, 1.0):
        assert P.cpu_cost(base, 77e3, 77e3) == P.gpu_cost(base, 77e3, 77e3)
    with pytest.raises(ValueError):
        P.cpu_cost(1.0, 0, 1)


def test_table_iii_base_costs():
    assert P.BASE_COST == {P.HASHAGG: 1.0, P.FILTER: 1.0, P.SHUFFLE: 1.0, P.PROJECT: 0.9,
                           P.HASHJOIN: 0.9, P.EXPAND: 0.9, P.SCAN: 0.8, P.SORT: 0.8}


def test_alg2_chain_examples():
    chain = [(P.SCAN, []), (P.FILTER, [0]), (P.PROJECT, [1])]
    assert P.map_device(chain, 15e3, 150e3) == [P.CPU] * 3
    assert P.map_device(chain, 1.5e6, 150e3) == [P.GPU] * 3
    # S:263 part == InfPT: middle op with a GPU predecessor: CPU = base + 0.1 > GPU = base -> GPU
    mid = [(P.SCAN, []), (P.FILTER, [0]), (P.PROJECT, [1]), (P.SORT, [2])]
    dev = P.map_device(mid, 150e3, 150e3)
    # Scan (first): GPU 0.8+0.1 > CPU 0.8 -> CPU; then Filter's predecessor is on the CPU
    assert dev[0] == P.CPU
    dev2 = P.map_device([(P.SCAN, []), (P.FILTER, [0])], 150e3 * 1.2, 150e3)
    assert dev2[0] == P.GPU


def test_alg2_traversal_children_first_left_to_right():
    assert P.traverse(P.DAGS["LR1"]) == [0, 1, 2, 3, 4]
    with pytest.raises(ValueError):
        P.traverse([(P.SCAN, [1]), (P.FILTER, [0])])                     # cycle


def test_alg2_extremes_every_catalog_dag():
    for name, dag in P.DAGS.items():
        for inf in (1e3, 150e3, 7e6):
            assert P.map_device(dag, inf * 10, inf) == [P.GPU] * len(dag), name
            assert P.map_device(dag, inf / 10, inf) == [P.CPU] * len(dag), name


def test_alg2_scale_invariance_and_monotonicity():
    rng = random.Random(2)
    for _ in range(1000):
        name = rng.choice(list(P.DAGS))
        part, inf = rng.uniform(1e3, 1e7), rng.uniform(1e3, 1e7)
        f = 2.0 ** rng.randrange(-10, 10)
        assert P.map_device(P.DAGS[name], part, inf) == P.map_device(P.DAGS[name], part * f, inf * f)
    # a single-op chain: GPU at size s => GPU at every s' > s
    for kind in P.BASE_COST:
        sizes = [150e3 * 1.05 ** e for e in range(-60, 60)]
        devs = [P.map_device([(kind, [])], s, 150e3)[0] for s in sizes]
        first_gpu = devs.index(P.GPU)
        assert all(d == P.GPU for d in devs[first_gpu:])


def test_alg2_matches_exhaustive_sequential_semantics_on_chains():
    # for a chain the greedy decision of op o depends only on o's predecessor's device:
    # check every op against the closed form of Eq. 7-9 with that predecessor fixed.
    for kinds in itertools.product(list(P.BASE_COST), repeat=3):
        chain = [(kinds[0], []), (kinds[1], [0]), (kinds[2], [1])]
        for part in (20e3, 100e3, 150e3, 200e3, 900e3):
            dev = P.map_device(chain, part, 150e3)
            for o, (k, preds) in enumerate(chain):
                x = part / 150e3
                c, gg, t = P.BASE_COST[k] * x, P.BASE_COST[k] / x, 0.1 * x
                if o in (0, 2) or dev[o - 1] == P.CPU:
                    gg += t
                else:
                    c += t
                assert dev[o] == (P.CPU if gg > c else P.GPU)


# ------------------------------------------------------------------ Eq. 10

def test_regression_recovers_exact_linear():
    rng = random.Random(7)
    rows = []
    for _ in range(10):
        thr, lat = rng.uniform(1, 100) * MB, rng.uniform(0.1, 10)
        rows.append((thr, lat, 100 + 2 * (thr / MB) - 3 * lat))
    b = G.fit(rows)
    assert b == pytest.approx((100, 2, -3), rel=1e-6)
    assert G.fit(rows[:2]) is None
    assert G.fit([(5 * MB, 1.0, 10.0)] * 5) is None                    # S:365 rank-deficient


def test_regression_targets_and_clamp():
    hist = [(2 * MB, 1.0, 0), (5 * MB, 2.0, 0), (3 * MB, 3.0, 0)]
    assert G.targets(hist, 5.0) == (5 * MB, 5.0)
    assert G.targets([(1, 2.0, 0), (1, 4.0, 0)], 0) == (1, 3.0)
    assert G.targets([(7, 1.5, 0)], 0) == (7, 1.5)
    assert G.predict((100e3, 0, 0), 123, 4) == 100e3
    assert G.predict((-5e3, 0, 0), 1, 1) == 1024.0
    assert G.predict((1e12, 0, 0), 1, 1) == 16 * 1024 * 1024


# ------------------------------------------------------------------ metrics

def test_nearest_rank():
    assert M.percentile_nearest_rank(range(1, 101), 99) == 99
    assert M.percentile_nearest_rank(range(1, 11), 99) == 10
    assert M.percentile_nearest_rank([4, 1, 3, 2], 50) == 2
    assert M.percentile_nearest_rank([5.0], 99) == 5.0
    assert M.avg_dataset_latency([(0.0, 2.0)]) == 2.0
    assert math.isclose(M.avg_dataset_latency([(0, 1), (1, 4)]), 2.0)
