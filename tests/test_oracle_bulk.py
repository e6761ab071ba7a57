"""Pins the column-form oracle (oracle/bulk.py, used by the 10M-record full-size checks) to
the brute-force oracle (oracle/queries.py, itself pinned to sqlite / hand-computed windows):
same rows, batch by batch, on streams small enough for brute force — including custom
windows, HAVING, ORDER BY ranks and the flush."""
import math

import pytest

import lmsgen as g
from lmsgen import vec
from oracle import bulk as B
from oracle import queries as Q


def _rows_by_key(rows):
    return {(r.win_start, r.key): r for r in rows}


@pytest.mark.parametrize("qname,traffic,secs,R,S,params", [
    ("LR2S", "B(0.6)", 47, None, None, g.LRParams(num_xways=2)),
    ("LR2S", "R(0.1,0.9)", 33, 6, 3, g.LRParams(num_xways=1)),
    ("CM2S", "B(0.5)", 70, None, None, g.CMParams(num_jobs=40)),
    ("CM2S", "U(0.4)", 25, 4, 2, g.CMParams(num_jobs=15, sel_ppm=600000)),
    ("CM1S", "B(0.3)", 75, None, None, g.CMParams()),
    ("CM1T", "R(0.2,0.5)", 130, None, None, g.CMParams()),
])
def test_bulk_matches_brute_force(qname, traffic, secs, R, S, params):
    q = Q.query_spec(qname, R, S)
    fam = q.family
    tr = g.Traffic.parse(traffic)
    data = list(g.stream_datasets(fam, tr, secs, seed=31, params=params))
    want = Q.replay(q, [[d] for _, d in data], num_xways=getattr(params, "num_xways", 10))
    rp = B.BulkReplay(q)
    got = []
    for t, _ in data:
        n = tr.count(t, 31)
        cols = vec.lr_columns(31, t, n, params) if fam == "LR" else vec.cm_columns(31, t, n, params)
        got.append(rp.batch(t, cols))
    got.append(rp.flush())
    assert len(got) == len(want)
    nonempty = 0
    for g_rows, w in zip(got, want):
        G, W = _rows_by_key(g_rows), _rows_by_key(w.rows)
        assert set(G) == set(W)
        nonempty += bool(W)
        for k, wr in W.items():
            gr = G[k]
            assert (gr.win_end, gr.count, gr.sum_fixed) == (wr.win_end, wr.count, wr.sum_fixed)
            assert math.isclose(gr.avg, wr.avg, rel_tol=1e-12) and math.isclose(gr.sum, wr.sum, rel_tol=1e-12)
            if qname == "LR2S":
                assert gr.avg == wr.avg and gr.sum == wr.sum      # integer sums: bit-exact
            if qname.startswith("CM1"):
                assert gr.rank == wr.rank
    assert nonempty >= 3


def _lr1_sorted(rows):
    return sorted((int(r["win_start"]), int(r["ts"]), int(r["vehicle"]), int(r["speed"]), int(r["xway"]),
                   int(r["lane"]), int(r["dir"]), int(r["seg"]), int(r["m"])) for r in rows)


@pytest.mark.parametrize("qname,traffic,secs,R,S,nveh,bsz", [
    ("LR1S", "B(0.2)", 47, None, None, 50, 5),          # Table IV LR1S, 5-second batches
    ("LR1S", "U(0.3)", 40, 18, 2, 40, 3),                # R/S = 9 panes per window
    ("LR1T", "R(0.1,0.4)", 75, None, None, 30, 7),      # tumbling: L = A
    ("LR1S", "B(0.1)", 30, 4, 1, 20, 1),
])
def test_bulk_lr1_matches_brute_force(qname, traffic, secs, R, S, nveh, bsz):
    """The column-form LR1 (vehicle counts per second -> window multiplicity m) equals the
    brute-force nested-loop self-join (queries.eval_instance, pinned to sqlite) batch by batch."""
    q = Q.query_spec(qname, R, S)
    tr = g.Traffic.parse(traffic)
    params = g.LRParams(num_vehicles=nveh)
    data = list(g.stream_datasets("LR", tr, secs, seed=43, params=params))
    batches = [data[i:i + bsz] for i in range(0, len(data), bsz)]
    want = Q.replay(q, [[d for _, d in b] for b in batches])
    rp = B.BulkLr1Replay(q)
    got = [rp.batch([(t, vec.lr_columns(43, t, tr.count(t, 43), params)) for t, _ in b]) for b in batches]
    got.append(rp.flush())
    assert len(got) == len(want)
    total = 0
    for gr, w in zip(got, want):
        assert _lr1_sorted(gr) == sorted((r.win_start, r.ts, r.vehicle, r.speed, r.xway, r.lane, r.dir, r.seg, r.m)
                                         for r in w.rows)
        total += len(gr)
    # every record is an L row of exactly one instance (its pane's), with m >= 1
    assert total == sum(tr.count(t, 43) for t, _ in data)
    assert all(int(x) >= 1 for b in got for x in b["m"])
