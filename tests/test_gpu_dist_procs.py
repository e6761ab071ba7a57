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
