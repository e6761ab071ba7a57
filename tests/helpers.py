"""Shared test helpers: drive the product through its binding and the oracle side by side."""
from __future__ import annotations

import math

import numpy as np

from oracle import queries as Q


def oracle_rows(qname, batches, num_xways=10, range_s=None, slide_s=None):
    q = Q.query_spec(qname, range_s, slide_s)
    return Q.replay(q, batches, num_xways=num_xways)


def product_run(qname, batches, flush=True, per_batch=True, device_batches=None, **cfg):
    """Push each batch's datasets (host memory), force a batch, sync; return per-batch outputs.

    device_batches: optional list parallel to batches with True for datasets that should be
    pushed through lms_push_device (torch CUDA buffers).
    """
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import _lib as L
    keep = []
    outs = []
    with P.Query(qname, mode="manual", **cfg) as q:
        t = 0.0
        for bi, b in enumerate(batches):
            for di, d in enumerate(b):
                if device_batches is not None and device_batches[bi][di]:
                    import torch
                    buf = torch.empty(len(d) + 64, dtype=torch.uint8, device="cuda")
                    buf[:len(d)].copy_(torch.frombuffer(bytearray(d), dtype=torch.uint8))
                    torch.cuda.synchronize()
                    keep.append(buf)
                    q.push_device(buf.data_ptr(), len(d), t)
                else:
                    q.push(d, t)
                t += 1.0
            q.force(t)
            st = q.sync(ok=(L.LMS_OK, L.LMS_EFORMAT))
            rec = q.record(q.num_batches() - 1)
            rows = q.read_lr1() if qname.upper().startswith("LR1") else q.read_agg()
            outs.append((rows, rec, st))
        if flush:
            st = q.flush(t, ok=(L.LMS_OK, L.LMS_EFORMAT))
            rec = q.record(q.num_batches() - 1)
            rows = q.read_lr1() if qname.upper().startswith("LR1") else q.read_agg()
            outs.append((rows, rec, st))
    return outs


def agg_key(qname, r):
    """Oracle AggRow key -> product key encoding."""
    if qname.upper() == "LR2S":
        x, d, s = r.key
        return (x * 2 + d) * 100 + s
    return r.key[0]


def compare_agg(qname, prod_rows: np.ndarray, ora_rows: list, rel=1e-9):
    """Element-by-element comparison of one batch's aggregate rows."""
    P = {}
    for r in prod_rows:
        k = (int(r["win_start_s"]), int(r["key"]))
        assert k not in P, f"duplicate product row {k}"
        P[k] = r
    O = {(r.win_start, agg_key(qname, r)): r for r in ora_rows}
    assert set(P) == set(O), (f"row keys differ: only product {sorted(set(P) - set(O))[:5]}, "
                              f"only oracle {sorted(set(O) - set(P))[:5]}")
    for k, o in O.items():
        p = P[k]
        assert int(p["win_end_s"]) == o.win_end
        assert int(p["count"]) == o.count, k
        assert int(p["sum_fixed"]) == o.sum_fixed, k
        if qname.upper() == "LR2S":
            # integer speed sums: SUM and AVG bit-exact
            assert float(p["sum"]) == o.sum and float(p["avg"]) == o.avg, k
            x, d, s = o.key
            assert (int(p["key_xway"]), int(p["key_dir"]), int(p["key_seg"])) == (x, d, s)
        else:
            assert math.isclose(float(p["sum"]), o.sum, rel_tol=rel, abs_tol=0), k
            assert math.isclose(float(p["avg"]), o.avg, rel_tol=rel, abs_tol=0), k
    if qname.upper() in ("CM1S", "CM1T"):
        # ORDER BY SUM(cpu): ranks must agree wherever sums differ by > 1e-9 relative (R9)
        by_win = {}
        for k, o in O.items():
            by_win.setdefault(k[0], []).append((o, P[k]))
        for rows in by_win.values():
            assert sorted(int(p["rank"]) for _, p in rows) == list(range(len(rows)))
            for o1, p1 in rows:
                for o2, p2 in rows:
                    if o1.sum < o2.sum and not math.isclose(o1.sum, o2.sum, rel_tol=1e-9):
                        assert int(p1["rank"]) < int(p2["rank"])


def compare_lr1(prod_rows: np.ndarray, ora_rows: list):
    got = sorted((int(r["win_start_s"]), int(r["ts"]), int(r["vehicle"]), int(r["speed"]), int(r["xway"]),
                  int(r["lane"]), int(r["dir"]), int(r["segment"]), int(r["multiplicity"])) for r in prod_rows)
    want = sorted((r.win_start, r.ts, r.vehicle, r.speed, r.xway, r.lane, r.dir, r.seg, r.m) for r in ora_rows)
    assert got == want


def compare_run(qname, prod_outs, ora_outs):
    assert len(prod_outs) == len(ora_outs)
    for (rows, rec, st), o in zip(prod_outs, ora_outs):
        if qname.upper().startswith("LR1"):
            compare_lr1(rows, o.rows)
        else:
            compare_agg(qname, rows, o.rows)
        assert rec["bad_records"] == o.bad, (rec["bad_records"], o.bad)
        assert rec["late_records"] == o.late, (rec["late_records"], o.late)
        assert rec["num_records"] == o.n_records
        assert rec["windows_closed"] == o.windows_closed, (rec["windows_closed"], o.windows_closed)
        assert rec["watermark"] == (-1 if o.watermark is None else o.watermark)
        assert rec["overflow_records"] == 0
