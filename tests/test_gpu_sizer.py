"""Sizer in the loop: lms_poll (Alg. 1 / CG(dN) / OS(tN)) on a virtual clock against the
oracle's Admission driver, and the query results of the batches it formed against the
oracle's windowed replay.

The product measures Proc for real on the GPU; the oracle mirror of the same 10 ms polling
loop (paper_2111_04289_b200/sim.py) is fed the product's measured Proc per batch (the
one input the oracle cannot know) and must then take the SAME decisions: same admit instants,
same dataset sets, same EstMaxLat (Eq. 6), same MaxLat (Eq. 5), same AvgThPut (Eq. 4).
"""
import math

import pytest

import lmsgen as g
from oracle import queries as Q
from oracle import sizer as Z
from tests.helpers import compare_agg, compare_lr1, oracle_rows

pytestmark = pytest.mark.gpu

REASON = {"bootstrap": 1, "slide": 2, "tumbling": 2, "tumbling-bootstrap": 3, "cap": 4, "trigger": 5,
          "forced": 0}


def oracle_mirror(mode, arrivals, t_end, procs, poll_s=0.01, slide_s=0.0, deadline_s=0.0, trigger_s=0.0):
    """sim.run's loop with oracle.sizer.Admission; procs[i] = measured Proc of batch i."""
    adm = Z.Admission(mode, slide_s=slide_s, deadline_s=deadline_s, trigger_s=trigger_s)
    out = []
    nxt, tick, last_tick = 0, 0, int(math.floor(t_end / poll_s + 1e-9))
    while tick <= last_tick:
        now = tick * poll_s
        while nxt < len(arrivals) and arrivals[nxt].ingest_s <= now + 1e-12:
            adm.push(Z.Dataset(nxt, arrivals[nxt].ingest_s, arrivals[nxt].nbytes))
            nxt += 1
        d = adm.poll(now)
        if not d.admitted:
            tick += 1
            continue
        i = len(out)
        thp_prev = adm.avg_thput
        maxlat = adm.complete(procs[i])
        out.append(dict(now=now, ids=[x.id for x in d.batch], est=d.est_max_lat, reason=d.reason,
                        max_lat=maxlat, avg_thput=adm.avg_thput, thp_prev=thp_prev))
        tick = max(tick + 1, int(math.ceil((now + procs[i]) / poll_s - 1e-9)))
    return out, tick


def check_run(qname, mode, traffic, seconds, parts, t_end, family=None, params=None, **cfg):
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import sim
    fam = family or qname[:2]
    secs = list(g.stream_datasets(fam, traffic, seconds, seed=77, params=params))
    arr = sim.split_seconds(fam, secs, parts)
    with P.Query(qname, mode=mode, **cfg) as q:
        res = sim.run(q, arr, t_end)
    recs = res.records
    assert len(recs) >= 3, "the run must form several batches"
    procs = [r["proc_s"] for r in recs]
    S = 0.0 if qname.endswith("T") else float(Q.query_spec(qname).slide_s)   # SlideTime
    ora, _ = oracle_mirror(mode, arr, t_end, procs, slide_s=S, deadline_s=cfg.get("deadline_s", 0.0),
                           trigger_s=cfg.get("trigger_s", 0.0))
    # ---- admission decisions (all but the final flush batch)
    assert len(ora) == len(recs) - 1
    for o, r, ids in zip(ora, recs, res.batches):
        assert r["admit_time_s"] == o["now"]
        assert ids == o["ids"]
        assert r["num_datasets"] == len(o["ids"])
        assert r["batch_bytes"] == sum(arr[i].nbytes for i in o["ids"])
        assert r["admit_reason"] == REASON[o["reason"]], (r["admit_reason"], o["reason"])
        if o["est"] is None:
            assert math.isnan(r["est_max_lat_s"])
        else:
            assert r["est_max_lat_s"] == pytest.approx(o["est"], rel=1e-12)
        assert r["max_lat_s"] == pytest.approx(o["max_lat"], rel=1e-12)
        assert r["avg_thput_Bps"] == pytest.approx(o["avg_thput"], rel=1e-12)
    assert res.batches[-1] == list(range(sum(len(b) for b in res.batches[:-1]), len(arr)))
    # ---- results of the formed batches == oracle replay of the same batches
    batches = [[arr[i].data for i in ids] for ids in res.batches]
    want = [o.rows for o in oracle_rows(qname, batches)]
    want[-2:] = [want[-2] + want[-1]]       # the product's flush batch carries the last datasets
    assert len(want) == len(res.rows)
    for rows, o in zip(res.rows, want):
        if qname.startswith("LR1"):
            compare_lr1(rows, o)
        else:
            compare_agg(qname, rows, o)
    return res, ora


def test_lmstream_sliding_lr2():
    """C3 shape (LR2S, R(L,U) traffic, Alg. 1 sliding branch: SlideTime = 10 s)."""
    res, ora = check_run("LR2S", "lmstream", "R(0.5,3)", 45, 4, 45.0)
    assert any(o["reason"] == "slide" for o in ora)
    # sliding admission: EstMaxLat reached SlideTime, and no earlier poll would have admitted
    for r in res.records[:-1]:
        if r["admit_reason"] == 2:
            assert r["est_max_lat_s"] >= 10.0 and r["max_buff_s"] < 10.0 + 0.011


def test_lmstream_tumbling_cm1t():
    """Tumbling branch (target = mean past MaxLat, Eq. 3 / R11)."""
    res, ora = check_run("CM1T", "lmstream", "U(1)", 40, 2, 40.0, params=g.CMParams(num_jobs=200))
    assert any(o["reason"] == "tumbling" for o in ora)


def test_lmstream_lr1s_u():
    """C2 shape (LR1S on U(N) traffic, SlideTime = 5 s)."""
    check_run("LR1S", "lmstream", "U(1.5)", 32, 3, 32.0)


def test_deadline_cg_d1_cm2():
    """CG(d1): Alg. 1 sliding branch with SlideTime := 1 s (reading R16), C5 shape."""
    res, ora = check_run("CM2S", "deadline", "B(2)", 20, 10, 20.0, deadline_s=1.0,
                         params=g.CMParams(num_jobs=500))
    assert sum(o["reason"] == "slide" for o in ora) >= 10


def test_deadline_cg_d0_lr2():
    """CG(d0): tumbling branch (mean past MaxLat)."""
    check_run("LR2S", "deadline", "B(1)", 20, 5, 20.0, deadline_s=0.0)


def test_trigger_os_t3_cm1s():
    """OS(t3): admit everything buffered at every 3 s trigger instant."""
    res, ora = check_run("CM1S", "trigger", "R(0.2,2)", 30, 2, 30.0, trigger_s=3.0)
    for o in ora:
        assert o["reason"] == "trigger"
        assert abs(o["now"] / 3.0 - round(o["now"] / 3.0)) < 1e-9


def test_percentiles_of_maxlat():
    """p50 / p99 MaxLat (nearest rank) through lms_percentile == oracle.metrics."""
    import ctypes as C

    from oracle.metrics import percentile_nearest_rank
    from paper_2111_04289_b200 import _lib as L
    res, _ = check_run("LR2S", "lmstream", "B(1)", 40, 4, 40.0)
    lat = [r["max_lat_s"] for r in res.records]
    arr = (C.c_double * len(lat))(*lat)
    for p in (50, 90, 99, 100):
        out = C.c_double()
        L.check(L.lms_percentile(arr, len(lat), p, C.byref(out)), "lms_percentile")
        assert out.value == percentile_nearest_rank(lat, p)


def test_online_infpt_regression_in_the_loop():
    """LMS_FLAG_ONLINE_INFPT: after every completed batch the library refits Eq. 10 on the
    (AvgThPut, MaxLat, InfPT) history and the next batch's Alg. 2 runs with the
    predicted InfPT — the oracle's exact-rational OLS on the same history must agree."""
    import paper_2111_04289_b200 as P
    from oracle import regression as RG
    from paper_2111_04289_b200 import _lib as L
    from paper_2111_04289_b200 import sim
    secs = list(g.stream_datasets("LR", "R(0.3,3)", 70, seed=9))
    arr = sim.split_seconds("LR", secs, 5)
    with P.Query("LR2S", mode="deadline", deadline_s=0.0, flags=L.LMS_FLAG_ONLINE_INFPT) as q:
        res = sim.run(q, arr, 70.0)
    recs = res.records
    assert len(recs) > 20
    hist, infpt, updates = [], 150e3, 0

    def conditioning(rows):
        """1 - corr^2 of the centred regressors (0: collinear)."""
        import numpy as np
        t = np.array([x[0] / 1e6 for x in rows]); lt = np.array([x[1] for x in rows])
        t, lt = t - t.mean(), lt - lt.mean()
        stt, sll, stl = (t * t).sum(), (lt * lt).sum(), (t * lt).sum()
        return 0.0 if stt <= 0 or sll <= 0 else 1.0 - stl * stl / (stt * sll)

    for r in recs:
        if r["inf_pt_bytes"] != pytest.approx(infpt, rel=1e-6):
            # fp vs exact-rational OLS may only part ways on a (near-)collinear history, where
            # Eq. 10's prediction is ill-posed; the feedback makes the runs differ after that
            assert len(hist) >= 3 and conditioning(hist[-256:]) < 1e-6, (len(hist), r["inf_pt_bytes"], infpt)
            break
        if r["num_datasets"] == 0:
            continue
        hist.append((r["avg_thput_Bps"], r["max_lat_s"], r["inf_pt_bytes"]))
        b = RG.fit(hist[-256:])
        if b is not None:
            infpt = RG.predict(b, *RG.targets(hist[-256:], 10.0))   # LR2S: SlideTime 10 s
            updates += 1
    assert updates > 10
    # the refit ran off the batch path: every batch after a refit carries its
    # duration, and the wait of the next launch on it (Table V "optimization blocking")
    fitted = [r for r in recs[1:] if r["opt_overhead_s"] > 0]
    assert len(fitted) > 10
    assert all(0 <= r["opt_block_s"] < 1.0 for r in recs)
    assert recs[0]["opt_overhead_s"] == 0 and recs[0]["opt_block_s"] == 0


@pytest.mark.parametrize("qname,fam,traffic", [("LR2S", "LR", "R(0.02,20)"), ("CM2S", "CM", "R(0.01,2)"),
                                              ("LR1S", "LR", "R(0.02,20)"), ("CM1S", "CM", "R(0.01,2)")])
def test_batch_plan_labels_match_oracle_planner(qname, fam, traffic):
    """Alg. 2 labels of every micro-batch (report-only): the record's plan_mask /
    n_cpu_ops / n_gpu_ops equal the oracle planner's MapDevice on the query's DAG with
    Part = batch bytes / NumCores and the batch's InfPT — batch sizes spanning the 150 KB
    inflection point (both device labels occur), also with the online Eq. 10 InfPT."""
    import paper_2111_04289_b200 as P
    from oracle import planner as PL
    from paper_2111_04289_b200 import _lib as L
    params = g.LRParams(num_vehicles=200) if qname == "LR1S" else None
    secs = [d for _, d in g.stream_datasets(fam, traffic, 40, seed=3, params=params)]
    sizes = [1, 1, 2, 5, 9, 13, 9]
    seen = set()
    for flags in (0, L.LMS_FLAG_ONLINE_INFPT):
        with P.Query(qname, mode="manual", flags=flags) as q:
            t, i = 0.0, 0
            for n in sizes:
                for d in secs[i:i + n]:
                    q.push(d, t)
                    t += 1.0
                i += n
                q.force(t)
                q.sync(ok=(L.LMS_OK, L.LMS_EFORMAT))
            recs = q.records()
        dag = PL.dag_for(qname)
        for r in recs:
            if r["batch_bytes"] == 0:
                continue
            want = PL.map_device(dag, r["batch_bytes"] / 12.0, r["inf_pt_bytes"], PL.BASE_TRANS_COST)
            mask = sum(1 << o for o, dv in enumerate(want) if dv == PL.GPU)
            assert r["plan_mask"] == mask, (r["batch_bytes"], r["inf_pt_bytes"], r["plan_mask"], want)
            assert r["n_gpu_ops"] == sum(1 for dv in want if dv == PL.GPU)
            assert r["n_cpu_ops"] == sum(1 for dv in want if dv == PL.CPU)
            seen.add(mask)
    assert len(seen) >= 2        # the sizes straddle the inflection point: both labellings occur
