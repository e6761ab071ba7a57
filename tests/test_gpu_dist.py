"""Multi-GPU protocol kernels on one GPU: G "virtual shard" handles (rank r of world G) each
get their record-boundary partition of every dataset; partial rows are bucketed by owner,
exchanged (LocalExchange: device copies) and merged by the owners.  The union of the owners'
rows must equal the single-stream oracle element by element (same comparator as the
single-GPU parity tests)."""
import pytest

import lmsgen as g
from tests.helpers import compare_agg, compare_lr1, oracle_rows

pytestmark = pytest.mark.gpu


def sharded_run(qname, batches, world, p2p=False, **cfg):
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200.dist import RankHandle, run_batch, split_points
    from tests.local_exchange import LocalExchange
    fam = qname[:2]
    hs = [RankHandle(P.Query(qname, mode="manual", rank=r, world=world, **cfg)) for r in range(world)]
    ex = LocalExchange()
    if p2p and p2p != "dense":
        ex.setup_p2p(hs, device_watermark=p2p == "device")
    outs, t = [], 0.0
    for b in batches + [None]:
        if b is not None:
            for d in b:
                for h, (o, n) in zip(hs, split_points(fam, d, world)):
                    if n:
                        h.q.push(d[o:o + n], t)
                t += 1.0
        run_batch(hs, ex, t, flush=b is None, p2p=p2p)
        rows = [h.q.read_lr1() if qname.startswith("LR1") else h.q.read_agg() for h in hs]
        recs = [h.q.record(h.q.num_batches() - 1) for h in hs]
        outs.append((rows, recs))
    for h in hs:
        h.q.close()
    return outs


@pytest.mark.parametrize("p2p", [False, True, "async", "device"], ids=["alltoall", "p2p", "p2p_async", "device"])
@pytest.mark.parametrize("qname,traffic,world", [("CM2S", "B(1.3)", 2), ("CM2S", "R(0.2,1.5)", 3),
                                                  ("LR2S", "B(1.7)", 2), ("LR2S", "U(0.8)", 4),
                                                  ("CM1S", "B(0.9)", 3), ("CM1T", "B(0.7)", 2)])
def test_virtual_shards_match_oracle(qname, traffic, world, p2p):
    import numpy as np
    fam = qname[:2]
    params = g.CMParams(num_jobs=300) if fam == "CM" else None
    secs = [d for _, d in g.stream_datasets(fam, traffic, 70 if qname != "CM1T" else 130, seed=21, params=params)]
    sizes = [4, 9, 1, 13, 6, 20]
    batches, i = [], 0
    for s in sizes:
        batches.append(secs[i:i + s])
        i += s
    batches.append(secs[i:])
    ora = oracle_rows(qname, batches)
    prod = sharded_run(qname, batches, world, p2p=p2p)
    assert len(prod) == len(ora)
    for (rows, recs), o in zip(prod, ora):
        compare_agg(qname, np.concatenate(rows), o.rows)
        assert sum(r["num_records"] for r in recs) == o.n_records
        assert sum(r["late_records"] for r in recs) == o.late
        assert all(r["windows_closed"] == o.windows_closed for r in recs)
        assert all(r["watermark"] == (-1 if o.watermark is None else o.watermark) for r in recs)


@pytest.mark.parametrize("qname,traffic,world", [("LR2S", "B(1.7)", 2), ("LR2S", "U(0.8)", 4),
                                                  ("CM1S", "B(0.9)", 3), ("CM1T", "B(0.7)", 2)])
def test_virtual_shards_dense_exchange(qname, traffic, world):
    """Dense exchange (small key sets): per merge window each rank's partial
    sums / counts as [instances][K] arrays, one SUM all-reduce, rank 0 finalizes — against
    the oracle (long flushes take several merge windows)."""
    test_virtual_shards_match_oracle(qname, traffic, world, "dense")


@pytest.mark.parametrize("qname,traffic,world", [("LR1S", "B(0.4)", 2), ("LR1S", "U(0.3)", 3), ("LR1T", "B(0.3)", 2)])
def test_virtual_shards_lr1_match_oracle(qname, traffic, world):
    """Multi-GPU LR1: every shard probes its own newest-slide rows against the all-reduced
    vehicle counts of the window; the union of the shards' rows (with multiplicities) equals
    the single-stream oracle's self-join."""
    import numpy as np
    params = g.LRParams(num_vehicles=150)          # many repeat vehicles: m > 1 is common
    secs = [d for _, d in g.stream_datasets("LR", traffic, 75, seed=23, params=params)]
    sizes = [4, 9, 1, 13, 6, 20]
    batches, i = [], 0
    for s in sizes:
        batches.append(secs[i:i + s])
        i += s
    batches.append(secs[i:])
    ora = oracle_rows(qname, batches)
    prod = sharded_run(qname, batches, world)
    assert len(prod) == len(ora)
    for (rows, recs), o in zip(prod, ora):
        compare_lr1(np.concatenate(rows), o.rows)
        assert sum(r["num_records"] for r in recs) == o.n_records
        assert all(r["windows_closed"] == o.windows_closed for r in recs)
        assert all(r["overflow_records"] == 0 for r in recs)
