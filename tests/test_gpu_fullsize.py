"""Full-size parity: BASELINE.json's 10M-record micro-batches, in bench.py's launch
configuration (one 10M-record dataset per second generated in HBM by lmsgen.cuda, borrowed
with lms_push_device, one MANUAL batch per second, then flush), checked element by element —
EVERY emitted row of every batch — against the column-form oracle (oracle/bulk.py) fed with
the same records' field columns (lmsgen.vec, pinned to the scalar generator).  Tolerance as
everywhere: keys / counts / exact sums bit-exact, CM SUM/AVG within 1e-9 relative."""
import pytest

import lmsgen as g
from lmsgen import vec
from oracle import bulk as B
from oracle import queries as Q
from tests.helpers import compare_agg

pytestmark = pytest.mark.gpu

N = 10_000_000


@pytest.mark.parametrize("qname,seconds", [("CM2S", 12), ("LR2S", 12), ("CM1S", 12)])
def test_full_size_batches_every_row(qname, seconds):
    import torch

    import paper_2111_04289_b200 as P
    from lmsgen import cuda as gcu
    fam = qname[:2]
    q = Q.query_spec(qname)
    rp = B.BulkReplay(q)
    seed = 211104289
    with P.Query(qname, mode="manual", max_batch_bytes=1 << 20) as dq:
        emitted = 0
        for t in range(seconds):
            buf, n = gcu.second_tensor(fam, t, N, seed=seed)
            dq.push_device(buf.data_ptr(), n, float(t))
            dq.force(float(t) + 1.0)
            dq.sync()
            rows = dq.read_agg()
            rec = dq.record(dq.num_batches() - 1)
            assert rec["num_records"] == N and rec["bad_records"] == 0 and rec["late_records"] == 0
            cols = vec.lr_columns(seed, t, N) if fam == "LR" else vec.cm_columns(seed, t, N)
            want = rp.batch(t, cols)
            compare_agg(qname, rows, want)
            emitted += len(want)
            del buf
            torch.cuda.empty_cache()
        dq.flush(float(seconds) + 1.0)
        rows = dq.read_agg()
        want = rp.flush()
        compare_agg(qname, rows, want)
        emitted += len(want)
    assert emitted > (20 if qname.startswith("CM1") else 1000)     # CM1: 4 categories per instance


def test_full_size_pipelined_as_bench_runs_it():
    """bench.py's exact configuration: 10M-record CM2 batches with LMS_FLAG_PIPELINE (batch i+1
    launched while batch i runs, rows read as batches complete); the union of all emitted rows
    equals the oracle's, row by row."""
    import numpy as np
    import torch

    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import _lib as L
    from lmsgen import cuda as gcu
    seconds, seed = 10, 211104289
    q = Q.query_spec("CM2S")
    rp = B.BulkReplay(q)
    want, got, live = [], [], []
    with P.Query("CM2S", mode="manual", max_batch_bytes=1 << 20, flags=L.LMS_FLAG_PIPELINE) as dq:
        for t in range(seconds):
            buf, n = gcu.second_tensor("CM", t, N, seed=seed)
            live.append(buf)                       # borrowed until its batch completes
            dq.push_device(buf.data_ptr(), n, float(t))
            dq.force(float(t) + 1.0)
            got.append(dq.read_agg())
            want += rp.batch(t, vec.cm_columns(seed, t, N))
            if len(live) > 3:
                live.pop(0)
        dq.sync()
        got.append(dq.read_agg())
        dq.flush(float(seconds) + 1.0)
        got.append(dq.read_agg())
        want += rp.flush()
        recs = dq.records()
    assert [r["num_records"] for r in recs[:seconds]] == [N] * seconds
    compare_agg("CM2S", np.concatenate(got), want)
    del live
    torch.cuda.empty_cache()
