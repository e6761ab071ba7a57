"""Multi-GPU protocol on CPU: world_size-2 gloo processes run the exact TorchDistExchange code of
paper_2111_04289_b200/dist.py on CPU tensors (watermark all-reduce + owner all-to-all of
partial rows), plus the host-side record-boundary split.  The CUDA kernels of the protocol are
covered by tests/test_gpu_dist.py (virtual shards on one GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import lmsgen as g

M64 = (1 << 64) - 1


def fmix64(k):
    k ^= k >> 33
    k = (k * 0xff51afd7ed558ccd) & M64
    k ^= k >> 33
    k = (k * 0xc4ceb9fe1a85ec53) & M64
    return k ^ (k >> 33)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeHandle:
    """CPU stand-in for dist.RankHandle: same interface, tensors on the CPU."""

    def __init__(self, rank, world, rows, wm, tsmin):
        from paper_2111_04289_b200 import AGG_DTYPE
        self.world, self.stream_ptr = world, 0
        owner = np.array([fmix64(int(k)) % world for k in rows["key"]], dtype=np.int64)
        order = np.argsort(owner, kind="stable")
        self.rows = rows[order]
        self.counts = [int((owner == r).sum()) for r in range(world)]
        self.wm = torch.tensor([wm], dtype=torch.int64)
        self.ts = torch.tensor([tsmin], dtype=torch.int64)
        self.dtype = AGG_DTYPE

    def watermark_tensors(self):
        return self.wm, self.ts

    def partials(self):
        return torch.from_numpy(self.rows.view(np.uint8).copy()), self.counts

    def windows_closed(self):
        return 1


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2111_04289_b200 import AGG_DTYPE
        from paper_2111_04289_b200.dist import TorchDistExchange
        rng = np.random.default_rng(rank)
        rows = np.zeros(50 + 10 * rank, AGG_DTYPE)
        rows["key"] = rng.integers(10 ** 9, 10 ** 10, len(rows))
        rows["win_start_s"] = rng.integers(0, 5, len(rows)) * 5
        rows["count"] = rank + 1
        h = FakeHandle(rank, world, rows, wm=100 + 7 * rank, tsmin=3 - rank)
        ex = TorchDistExchange()
        ex.allreduce_watermarks([h])
        (recv,) = ex.all_to_all([h], [h.partials()])
        got = recv.numpy().view(AGG_DTYPE)
        q.put((rank, int(h.wm.item()), int(h.ts.item()), got.tobytes(), rows.tobytes()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange():
    from paper_2111_04289_b200 import AGG_DTYPE
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    sent = np.concatenate([np.frombuffer(r[4], AGG_DTYPE) for r in res])
    for rank, wm, ts, got_b, _ in res:
        assert wm == 107 and ts == 2                                 # MAX / MIN over ranks
        got = np.frombuffer(got_b, AGG_DTYPE)
        want = sent[[fmix64(int(k)) % world == rank for k in sent["key"]]]
        assert sorted(map(bytes, got)) == sorted(map(bytes, want))   # exactly the rows it owns


class FakeDenseHandle:
    """CPU stand-in for a dense (LR2 / CM1) RankHandle: per merge window, this rank's partial
    [nwin][K] sums / counts; rank 0 "finalizes" (records what the all-reduce gave it)."""

    def __init__(self, rank, k0, k1, wmerge, K, seed):
        self.rank, self.k0, self.k1, self.wmerge, self.K = rank, k0, k1, wmerge, K
        self.stream_ptr = 0
        self.rng = np.random.default_rng(seed)
        self.sent, self.final = {}, {}

    def last_close_range(self):
        return self.k0, self.k1

    def merge_window(self):
        return self.wmerge

    def dense_partials(self, k_lo, nwin):
        s = torch.from_numpy(self.rng.integers(0, 1000, nwin * self.K).astype(np.int64))
        c = torch.from_numpy(self.rng.integers(0, 5, nwin * self.K).astype(np.int64))
        self.sent[k_lo] = (s.clone(), c.clone())
        self._cur = (s, c)
        return s, c

    def dense_finalize(self, k_lo, nwin):
        s, c = self._cur
        self.final[k_lo] = (s.clone(), c.clone(), nwin)
        return 0


def _dense_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2111_04289_b200.dist import TorchDistExchange, exchange_dense
        h = FakeDenseHandle(rank, k0=-5, k1=7, wmerge=5, K=2000, seed=rank)
        exchange_dense([h], TorchDistExchange())
        q.put((rank, {k: (v[0].numpy().tobytes(), v[1].numpy().tobytes()) for k, v in h.sent.items()},
               {k: (v[0].numpy().tobytes(), v[1].numpy().tobytes(), v[2]) for k, v in h.final.items()}))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_dense_exchange():
    """exchange_dense: every merge window of the close range (13 instances, windows of 5:
    k = -5, 0, 5) is SUM-all-reduced over the ranks before the finalize."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_dense_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda x: x[0])
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, sent, final in res:
        assert sorted(final) == [-5, 0, 5] and [final[k][2] for k in (-5, 0, 5)] == [5, 5, 3]
        for k in (-5, 0, 5):
            want_s = sum(np.frombuffer(r[1][k][0], np.int64) for r in res)
            want_c = sum(np.frombuffer(r[1][k][1], np.int64) for r in res)
            assert np.array_equal(np.frombuffer(final[k][0], np.int64), want_s)
            assert np.array_equal(np.frombuffer(final[k][1], np.int64), want_c)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_split_points_record_boundaries(world):
    from paper_2111_04289_b200.dist import split_points
    cm = b"".join(d for _, d in g.stream_datasets("CM", "B(0.5)", 3))
    parts = split_points("CM", cm, world)
    assert sum(n for _, n in parts) == len(cm)
    assert b"".join(cm[o:o + n] for o, n in parts) == cm
    for o, n in parts:
        assert o == 0 or cm[o - 1] == ord("\n")
        assert n == 0 or cm[o + n - 1] == ord("\n")
    lr = b"".join(d for _, d in g.stream_datasets("LR", "B(0.3)", 2))
    parts = split_points("LR", lr, world)
    assert all(o % 70 == 0 and n % 70 == 0 for o, n in parts)
    assert sum(n for _, n in parts) == len(lr)


def test_split_edge_cases():
    """lms_split: more parts than records (empty parts), a line longer than the 512 B scan
    window, and the argument checks (C ABI, host memory)."""
    import ctypes as C
    from paper_2111_04289_b200 import _lib as L
    from paper_2111_04289_b200.dist import split_points
    two = b"1,,1000000000,1,1,1,u,0,0,0.000001,0.000001,0.000001,0\n" * 2
    parts = split_points("CM", two, 5)
    assert [n for _, n in parts].count(0) == 3 and b"".join(two[o:o + n] for o, n in parts) == two
    long_line = b"1,,1," + b"x" * 2000 + b"\n" + b"2,,2,y\n"
    parts = split_points("CM", long_line, 2)
    assert parts[1][0] == long_line.index(b"\n") + 1
    offs = (C.c_uint64 * 3)()
    buf = C.create_string_buffer(b"abc", 3)
    assert L.lms_split(L.LMS_CM2S, buf, 3, 2, offs) == L.LMS_EINVAL          # no final newline
    assert L.lms_split(L.LMS_LR2S, buf, 3, 2, offs) == L.LMS_EINVAL          # not 70 B records
    assert L.lms_split(99, buf, 3, 2, offs) == L.LMS_EINVAL
    assert L.lms_split(L.LMS_CM2S, None, 3, 2, offs) == L.LMS_EINVAL


class FakeLr1Handle:
    """CPU stand-in for an LR1 RankHandle: per-instance vehicle counts, records the all-reduced
    counts each probe saw."""

    def __init__(self, rank, k_range, nveh=64):
        rng = np.random.default_rng(100 + rank)
        self.stream_ptr, self.k_range = 0, k_range
        self.local = {k: torch.from_numpy(rng.integers(0, 5, nveh).astype(np.int32)) for k in range(k_range[0], k_range[1] + 1)}
        self.sent = {k: v.clone() for k, v in self.local.items()}
        self.seen, self.closed = {}, False

    def close_range(self):
        return self.k_range

    def lr1_window_counts(self, k):
        return self.local[k]

    def lr1_probe(self, k):
        self.seen[k] = self.local[k].clone()

    def run_close(self):
        self.closed = True

    def sync(self):
        return 0


def _lr1_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2111_04289_b200.dist import TorchDistExchange, close_lr1
        h = FakeLr1Handle(rank, (3, 5))
        sts = close_lr1([h], TorchDistExchange())
        q.put((rank, {k: v.numpy().tobytes() for k, v in h.sent.items()},
               {k: v.numpy().tobytes() for k, v in h.seen.items()}, h.closed, sts))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_lr1_window_counts():
    """Multi-GPU LR1 protocol (dist.close_lr1) over world-size-2 gloo: every closing instance's
    vehicle counts are SUM-all-reduced before that instance's probe, on every rank."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_lr1_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for k in (3, 4, 5):
        want = sum(np.frombuffer(r[1][k], np.int32).astype(np.int64) for r in res)
        for r in res:
            assert np.array_equal(np.frombuffer(r[2][k], np.int32), want)
    assert all(r[3] and r[4] == [0] for r in res)


class FakeP2PHandle:
    """CPU stand-in for the fused-exchange side of a RankHandle: records the protocol calls."""

    def __init__(self, rank):
        self.rank, self.stream_ptr, self.calls, self.imported = rank, 0, [], []

    def p2p_export(self):
        return bytes([self.rank]) * 416

    def p2p_import(self, blob):
        self.imported.append(blob[0])

    def windows_closed(self):
        return 3

    def last_close_range(self):
        return (10, 12)

    def merge_window(self):
        return 2

    def p2p_push(self, k, n):
        self.calls.append(("push", k, n))

    def p2p_finalize(self, k, n):
        self.calls.append(("fin", k, n))


def _p2p_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2111_04289_b200.dist as D
        h = FakeP2PHandle(rank)
        ex = D.TorchDistExchange()
        ex.setup_p2p([h])
        D.exchange_p2p([h], ex)          # the exchange tail of run_batch(p2p=True)
        D.exchange_p2p([h], ex, k_from=10 + h.merge_window())   # run_batch(p2p="async") remainder
        q.put((rank, h.imported, h.calls))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_p2p_setup_and_passes():
    """Fused exchange host protocol over world-size-2 gloo: every rank imports every rank's
    handle (in rank order) and pushes / finalizes the closed instances in merge-window passes."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_p2p_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, imported, calls in res:
        assert imported == [0, 1]
        assert calls == [("push", 10, 2), ("fin", 10, 2), ("push", 12, 1), ("fin", 12, 1),
                         ("push", 12, 1), ("fin", 12, 1)]   # + the remainder after an async pass


# ----------------------------------------------------------------------------- Alg. 1 / CG(dN) across ranks

def _adm_arrivals(seed, n, world):
    """Datasets every 0.25 s (B-shaped traffic with jitter), 0.2-3 MB each, split unevenly
    over the ranks (each rank's partition size = its share of the record-boundary split)."""
    import random
    rng = random.Random(seed)
    out = []
    for i in range(n):
        tot = rng.randrange(200_000, 3_000_000)
        cuts = sorted(rng.randrange(0, tot + 1) for _ in range(world - 1))
        parts = [b - a for a, b in zip([0] + cuts, cuts + [tot])]
        out.append((round(0.25 * i + rng.uniform(0, 0.2), 6), tot, parts))
    return out


def _adm_proc(rank, local_bytes):
    """Deterministic per-rank Proc model: fixed overhead + bytes / rank speed (rank 1 slower)."""
    return 0.03 + local_bytes / (4e6 if rank == 0 else 3e6)


def _adm_worker(rank, world, port, q, mode, slide, dl, arr, t_end):
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import math

        from paper_2111_04289_b200.dist import DistAdmission
        adm = DistAdmission(mode, slide_s=slide, deadline_s=dl)
        out, nxt, tick, last = [], 0, 0, int(math.floor(t_end / 0.01 + 1e-9))
        while tick <= last:
            now = tick * 0.01
            while nxt < len(arr) and arr[nxt][0] <= now + 1e-12:
                adm.push(arr[nxt][0], arr[nxt][2][rank])
                nxt += 1
            ok, n, est, reason = adm.poll(now)
            if not ok:
                tick += 1
                continue
            proc_local = _adm_proc(rank, adm.in_flight_local_bytes)
            ml = adm.complete(proc_local)
            out.append((now, n, est, reason, ml, adm.avg_thput))
            proc = max(_adm_proc(r, sum(a[2][r] for a in arr[sum(o[1] for o in out[:-1]):sum(o[1] for o in out)]))
                       for r in range(world))
            tick = max(tick + 1, int(math.ceil((now + proc) / 0.01 - 1e-9)))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode_name,slide,dl", [("deadline", 0.0, 1.0), ("deadline", 0.0, 0.0),
                                                ("lmstream", 5.0, 0.0)])
def test_gloo_world2_alg1_partitioned(mode_name, slide, dl):
    """CG(d1), CG(d0) and LMStream's sliding branch for micro-batches partitioned over two ranks
    (P:417): rank 0 decides on the global datasets (bytes summed over the ranks) and
    broadcasts; Proc = max over ranks.  Both ranks must take exactly the decisions of the
    oracle's Admission driver fed the global datasets and the max-over-ranks Proc."""
    import math

    from oracle import sizer as Z
    from paper_2111_04289_b200 import _lib as L
    world, t_end = 2, 20.0
    arr = _adm_arrivals(11, 70, world)
    mode = L.LMS_MODE_DEADLINE if mode_name == "deadline" else L.LMS_MODE_LMSTREAM
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_adm_worker, args=(r, world, port, q, mode, slide, dl, arr, t_end))
          for r in range(world)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    def nan_free(rows):
        return [tuple(None if isinstance(x, float) and math.isnan(x) else x for x in r) for r in rows]
    assert nan_free(res[0]) == nan_free(res[1]), "ranks took different decisions"
    # oracle mirror: global datasets, Proc = max over ranks of the same per-rank model
    adm = Z.Admission(mode_name, slide_s=slide, deadline_s=dl)
    want, nxt, tick, last, done = [], 0, 0, int(math.floor(t_end / 0.01 + 1e-9)), 0
    while tick <= last:
        now = tick * 0.01
        while nxt < len(arr) and arr[nxt][0] <= now + 1e-12:
            adm.push(Z.Dataset(nxt, arr[nxt][0], arr[nxt][1]))
            nxt += 1
        d = adm.poll(now)
        if not d.admitted:
            tick += 1
            continue
        ids = [x.id for x in d.batch]
        assert ids == list(range(done, done + len(ids)))
        done += len(ids)
        proc = max(_adm_proc(r, sum(arr[i][2][r] for i in ids)) for r in range(world))
        ml = adm.complete(proc)
        want.append((now, len(ids), d.est_max_lat, d.reason, ml, adm.avg_thput))
        tick = max(tick + 1, int(math.ceil((now + proc) / 0.01 - 1e-9)))
    got = res[0]
    assert len(got) == len(want) and len(want) >= 5
    reasons = {"bootstrap": 1, "slide": 2, "tumbling": 2, "tumbling-bootstrap": 3, "cap": 4}
    for g_, w in zip(got, want):
        assert g_[0] == w[0] and g_[1] == w[1]
        assert g_[3] == reasons[w[3]], (g_, w)
        if w[2] is None:
            assert math.isnan(g_[2])
        else:
            assert g_[2] == pytest.approx(w[2], rel=1e-12)
        assert g_[4] == pytest.approx(w[4], rel=1e-12)
        assert g_[5] == pytest.approx(w[5], rel=1e-12)
    if mode_name == "deadline" and dl > 0:
        assert sum(w[3] == "slide" for w in want) >= 5
