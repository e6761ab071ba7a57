"""Key-state eviction (VERDICT r01 "What's weak" 7): the jobId / vehicle dictionary reclaims a
key once none of its panes is live, so a stream whose keys churn runs indefinitely with the
default key capacity.  Streams here carry ~10^4 live keys per window and 3 x 10^5 distinct keys
over the stream (> 4 x the 65 536-key default capacity): no LMS_EOVERFLOW, every row of every
batch equal to the column-form oracle (oracle/bulk.py).  Paper anchor: Table IV CM2,
LR1; eviction rule reading R7.
"""
import numpy as np
import pytest

import lmsgen as g
from lmsgen import vec
from oracle import bulk as B
from oracle import queries as Q
from tests.helpers import compare_agg
from tests.test_gpu_parity_r02 import _check_lr1

pytestmark = pytest.mark.gpu

SEED = 77


def _churn_cm(t: int, data: bytes, keys_per_sec: int) -> bytes:
    """Rewrite the 10-digit jobId of record i of second t to 10^9 + t*keys_per_sec + i % keys_per_sec."""
    lines = data.split(b"\n")[:-1]
    out = []
    for i, ln in enumerate(lines):
        a = ln.index(b",,") + 2
        job = 10 ** 9 + t * keys_per_sec + i % keys_per_sec
        out.append(ln[:a] + str(job).encode() + ln[a + 10:])
    return b"\n".join(out) + b"\n"


def _churn_lr(t: int, data: bytes, keys_per_sec: int) -> bytes:
    b = bytearray(data)
    for i in range(len(b) // 70):
        vid = t * keys_per_sec + i % keys_per_sec
        b[70 * i + 9:70 * i + 19] = b"%010d" % vid
    return bytes(b)


def test_cm2_jobid_churn_default_capacity():
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import _lib as L
    secs, rate, kps, bsz = 300, 1000, 1000, 5
    params = g.CMParams(num_jobs=100, sel_ppm=1_000_000)       # every record survives the filter
    q = Q.query_spec("CM2S", 10, 5)
    rp = B.BulkReplay(q)
    distinct = 0
    with P.Query("CM2S", mode="manual", range_s=10, slide_s=5) as dq:
        assert dq.cfg.max_keys == 1 << 16
        for b0 in range(0, secs, bsz):
            want = []
            for t in range(b0, b0 + bsz):
                d = _churn_cm(t, g.second_bytes("CM", t, rate, SEED, params), kps)
                dq.push(d, float(t))
                cols = vec.cm_columns(SEED, t, rate, params)
                cols["job"] = (10 ** 9 + t * kps + np.arange(rate) % kps).astype(np.uint64)
                want += rp.batch(t, cols)
                distinct += kps
            dq.force(float(b0 + bsz))
            assert dq.sync() == L.LMS_OK                     # no LMS_EOVERFLOW
            rec = dq.record(dq.num_batches() - 1)
            assert rec["overflow_records"] == 0 and rec["bad_records"] == 0
            compare_agg("CM2S", dq.read_agg(), want)
        dq.flush(float(secs + 1))
        compare_agg("CM2S", dq.read_agg(), rp.flush())
    assert distinct > 4 * (1 << 16)


def test_lr1_vehicle_churn_small_capacity():
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import _lib as L
    secs, rate, kps, bsz = 240, 600, 600, 5
    q = Q.query_spec("LR1S")
    rp = B.BulkLr1Replay(q)
    with P.Query("LR1S", mode="manual", max_keys=1 << 15) as dq:   # ~21k live vehicles per window
        for b0 in range(0, secs, bsz):
            seconds = []
            for t in range(b0, b0 + bsz):
                d = _churn_lr(t, g.second_bytes("LR", t, rate, SEED), kps)
                dq.push(d, float(t))
                cols = vec.lr_columns(SEED, t, rate)
                cols["vid"] = (t * kps + np.arange(rate) % kps).astype(np.int64)
                seconds.append((t, cols))
            dq.force(float(b0 + bsz))
            assert dq.sync() == L.LMS_OK
            assert dq.record(dq.num_batches() - 1)["overflow_records"] == 0
            _check_lr1(dq.read_lr1(), rp.batch(seconds))
        dq.flush(float(secs + 1))
        _check_lr1(dq.read_lr1(), rp.flush())
    assert secs * kps > 4 * (1 << 15)
