"""Multi-process parity: 2 ranks (separate processes, as under torchrun) each own an lms_query
(rank r of world 2), push their record-boundary partition of every dataset, and run the
dist.py protocol with TorchDistExchange (gloo with host staging, since the test box has one
GPU).  The union of the owners' rows must equal the single-stream oracle, batch by batch."""
import os
import socket

import numpy as np
import pytest

import lmsgen as g
from tests.helpers import compare_agg, compare_lr1, oracle_rows

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, qname, batches, out_q, p2p=False):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2111_04289_b200 as P
        from paper_2111_04289_b200.dist import RankHandle, TorchDistExchange, run_batch, split_points
        h = RankHandle(P.Query(qname, mode="manual", rank=rank, world=world))
        ex = TorchDistExchange()
        if p2p:
            ex.setup_p2p([h], device_watermark=p2p == "device")   # CUDA IPC mappings
        t, outs = 0.0, []
        for b in batches + [None]:
            if b is not None:
                for d in b:
                    o, n = split_points(qname[:2], d, world)[rank]
                    if n:
                        h.q.push(d[o:o + n], t)
                    t += 1.0
            run_batch([h], ex, t, flush=b is None, p2p=p2p)
            rec = h.q.record(h.q.num_batches() - 1)
            rows = h.q.read_lr1() if qname.startswith("LR1") else h.q.read_agg()
            outs.append((rows.tobytes(), rec["num_records"], rec["windows_closed"]))
        h.q.close()
        out_q.put((rank, outs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("qname,traffic,p2p", [("CM2S", "B(1.5)", False), ("LR2S", "R(0.5,2)", False),
                                               ("CM1S", "B(0.8)", False), ("LR1S", "B(0.4)", False),
                                               ("CM2S", "B(1.5)", True), ("LR2S", "R(0.5,2)", True),
                                               ("CM1S", "B(0.8)", True), ("CM2S", "B(1.5)", "async"),
                                               ("LR2S", "R(0.5,2)", "async"), ("CM2S", "B(1.5)", "device"),
                                               ("CM1S", "B(0.8)", "device")])
def test_two_processes_match_oracle(qname, traffic, p2p):
    import torch.multiprocessing as mp
    from paper_2111_04289_b200 import AGG_DTYPE, LR1_DTYPE
    fam = qname[:2]
    params = g.CMParams(num_jobs=200) if fam == "CM" else (g.LRParams(num_vehicles=150) if qname == "LR1S" else None)
    secs = [d for _, d in g.stream_datasets(fam, traffic, 75, seed=5, params=params)]
    batches = [secs[i:i + 7] for i in range(0, len(secs), 7)]
    ora = oracle_rows(qname, batches)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_main, args=(r, 2, port, qname, batches, q, p2p)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(2))
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert len(res[0]) == len(res[1]) == len(ora)
    for i, o in enumerate(ora):
        dt = LR1_DTYPE if qname.startswith("LR1") else AGG_DTYPE
        rows = np.concatenate([np.frombuffer(res[r][i][0], dt) for r in range(2)])
        if qname.startswith("LR1"):
            compare_lr1(rows, o.rows)
        else:
            compare_agg(qname, rows, o.rows)
        assert res[0][i][1] + res[1][i][1] == o.n_records
        assert res[0][i][2] == res[1][i][2] == o.windows_closed


def _rank_cg(rank, world, port, qname, arrivals, t_end, deadline, out_q):
    """CG(dN) across processes: DistAdmission decides (rank 0, broadcast) on a 10 ms virtual
    poll clock, each rank pushes its partition of every arrival and forces it when admitted;
    the batch's measured Proc of every rank feeds complete() (max over ranks)."""
    import math

    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2111_04289_b200 as P
        from paper_2111_04289_b200 import _lib as L
        from paper_2111_04289_b200.dist import (DistAdmission, RankHandle, TorchDistExchange, run_batch,
                                                split_points)
        h = RankHandle(P.Query(qname, mode="manual", rank=rank, world=world))
        ex = TorchDistExchange()
        adm = DistAdmission(L.LMS_MODE_DEADLINE, deadline_s=deadline)
        dec, outs, nxt, tick = [], [], 0, 0
        last = int(math.floor(t_end / 0.01 + 1e-9))
        while tick <= last:
            now = tick * 0.01
            while nxt < len(arrivals) and arrivals[nxt][0] <= now + 1e-12:
                ing, d = arrivals[nxt]
                o, n = split_points(qname[:2], d, world)[rank]
                if n:
                    h.q.push(d[o:o + n], ing)
                adm.push(ing, n)
                nxt += 1
            ok, n_ds, est, reason = adm.poll(now)
            if not ok:
                tick += 1
                continue
            run_batch([h], ex, now)
            rec = h.q.record(h.q.num_batches() - 1)
            ml = adm.complete(rec["proc_s"])
            rows = h.q.read_agg()
            dec.append((now, n_ds, est, reason, ml, adm.avg_thput, adm.last_proc))
            outs.append((rows.tobytes(), rec["num_records"]))
            tick = max(tick + 1, int(math.ceil((now + adm.last_proc) / 0.01 - 1e-9)))
        run_batch([h], ex, t_end + 1.0, flush=True)         # remaining datasets + final windows
        outs.append((h.q.read_agg().tobytes(), h.q.record(h.q.num_batches() - 1)["num_records"]))
        h.q.close()
        out_q.put((rank, dec, outs, nxt))
    finally:
        dist.destroy_process_group()


def test_two_processes_deadline_cg_d1():
    """CG(d1) (Alg. 1 sliding branch, SlideTime := 1 s, reading R16) for micro-batches
    partitioned over two processes: both ranks take the decisions of the oracle's
    Admission driver fed the global datasets and the max-over-ranks measured Proc (same admit
    instants, dataset counts, EstMaxLat, MaxLat, AvgThPut), and the union of the ranks' rows of
    every formed batch equals the oracle's replay of the same batches."""
    import math

    import torch.multiprocessing as mp
    from oracle import sizer as Z
    from paper_2111_04289_b200 import AGG_DTYPE
    from paper_2111_04289_b200 import sim
    qname, t_end, deadline = "CM2S", 20.0, 1.0
    secs = list(g.stream_datasets("CM", "B(2)", 20, seed=31, params=g.CMParams(num_jobs=300)))
    arr = [(a.ingest_s, bytes(a.data)) for a in sim.split_seconds("CM", secs, 8)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_cg, args=(r, 2, port, qname, arr, t_end, deadline, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = {r: (d, o, n) for r, d, o, n in (q.get(timeout=600) for _ in range(2))}
    for p in ps:
        p.join(timeout=120)
        assert p.exitcode == 0
    dec0, dec1 = res[0][0], res[1][0]
    assert [x[:2] + x[3:] for x in dec0] == [x[:2] + x[3:] for x in dec1]
    assert len(dec0) >= 10
    # ---- oracle mirror: global datasets, the measured max-over-ranks Proc
    adm = Z.Admission("deadline", deadline_s=deadline)
    batches, nxt, tick, k = [], 0, 0, 0
    last = int(math.floor(t_end / 0.01 + 1e-9))
    while tick <= last:
        now = tick * 0.01
        while nxt < len(arr) and arr[nxt][0] <= now + 1e-12:
            adm.push(Z.Dataset(nxt, arr[nxt][0], len(arr[nxt][1])))
            nxt += 1
        d = adm.poll(now)
        if not d.admitted:
            tick += 1
            continue
        got = dec0[k]
        proc = got[6]
        assert got[0] == now and got[1] == len(d.batch)
        if d.est_max_lat is None:
            assert math.isnan(got[2])
        else:
            assert got[2] == pytest.approx(d.est_max_lat, rel=1e-12)
        ml = adm.complete(proc)
        assert got[4] == pytest.approx(ml, rel=1e-12)
        assert got[5] == pytest.approx(adm.avg_thput, rel=1e-12)
        batches.append([arr[x.id][1] for x in d.batch])
        k += 1
        tick = max(tick + 1, int(math.ceil((now + proc) / 0.01 - 1e-9)))
    assert k == len(dec0)
    assert sum(1 for x in dec0 if x[3] == 2) >= 5            # slide admissions (EstMaxLat >= 1 s)
    # ---- results: formed batches (+ the flush batch carrying the rest) vs the oracle replay
    rest = [arr[i][1] for i in range(sum(len(b) for b in batches), res[0][2])]
    ora = oracle_rows(qname, batches + [rest])
    outs0, outs1 = res[0][1], res[1][1]
    assert len(outs0) == len(outs1) == len(batches) + 1
    assert len(ora) == len(batches) + 2                     # + the rest batch + the final flush
    want = [o.rows for o in ora[:len(batches)]] + [np.concatenate([ora[-2].rows, ora[-1].rows])]
    for i, w in enumerate(want):
        rows = np.concatenate([np.frombuffer(outs0[i][0], AGG_DTYPE), np.frombuffer(outs1[i][0], AGG_DTYPE)])
        compare_agg(qname, rows, w)
