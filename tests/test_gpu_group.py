"""Single-handle multi-device driver (lms_config.num_gpus / device_ids):
one lms_query row-partitions every micro-batch over G devices, merges the partial aggregates
by key owner through peer memory, and sizes batches with Alg. 1 / CG(dN) on the whole batch.
On the one-GPU test box the G "devices" are the same ordinal (virtual shards: the same
kernels, peer pointers that happen to be local).  Every row against the oracle; the sizer
decisions against the oracle's Admission driver fed the measured Proc (as test_gpu_sizer).
"""
import pytest

import lmsgen as g
from tests.helpers import compare_run, oracle_rows, product_run
from tests.test_gpu_sizer import check_run

pytestmark = pytest.mark.gpu


def stream(family, traffic, seconds, seed=13, params=None):
    return [d for _, d in g.stream_datasets(family, traffic, seconds, seed=seed, params=params)]


@pytest.mark.parametrize("qname,traffic,secs,bs,G", [
    ("CM2S", "B(1.3)", 40, [5, 5, 1, 9, 2], 2),
    ("CM2S", "R(0.2,1)", 33, [7, 7, 7], 3),
    ("LR2S", "B(1.7)", 45, [3, 7, 1, 10, 4], 2),
    ("CM1S", "B(0.9)", 75, [10, 10, 3, 20], 2),
    ("CM1T", "U(0.5)", 130, [30, 30, 60], 4),
    ("LR1S", "B(0.4)", 40, [5, 5, 2, 8], 2),
    ("LR1T", "B(0.3)", 65, [7, 11, 30], 3),
])
def test_group_parity_streams(qname, traffic, secs, bs, G):
    fam = qname[:2]
    params = g.LRParams(num_vehicles=300) if qname.startswith("LR1") else (
        g.CMParams(num_jobs=200) if fam == "CM" else None)
    data = stream(fam, traffic, secs, params=params)
    batches, i = [], 0
    for n in bs:
        batches.append(data[i:i + n])
        i += n
    if i < len(data):
        batches.append(data[i:])
    compare_run(qname, product_run(qname, batches, device_ids=[0] * G), oracle_rows(qname, batches))


def test_group_device_pushes_and_long_flush():
    """Device-resident datasets (each device's part staged or borrowed) and a close emitting
    more instances than one merge window (host-driven exchange passes)."""
    data = stream("CM", "B(0.4)", 36, params=g.CMParams(num_jobs=50))
    batches = [data[:30], data[30:]]
    devmask = [[i % 2 == 0 for i in range(len(b))] for b in batches]
    for qname in ("CM2S", "CM1S"):
        compare_run(qname, product_run(qname, batches, device_batches=devmask, device_ids=[0, 0],
                                       range_s=4, slide_s=1),
                    oracle_rows(qname, batches, range_s=4, slide_s=1))
    lr = stream("LR", "B(0.5)", 30)
    compare_run("LR2S", product_run("LR2S", [lr[:25], lr[25:]], device_ids=[0, 0, 0], range_s=3, slide_s=1),
                oracle_rows("LR2S", [lr[:25], lr[25:]], range_s=3, slide_s=1))


def test_group_alg1_deadline_cg_d1():
    """CG(d1) (reading R16) sizing the whole micro-batch of a 2-device handle: same admit
    instants / dataset sets / Eq. 4-6 values as the oracle fed the measured Proc."""
    res, ora = check_run("CM2S", "deadline", "B(2)", 20, 10, 20.0, deadline_s=1.0,
                         params=g.CMParams(num_jobs=500), device_ids=[0, 0])
    assert sum(o["reason"] == "slide" for o in ora) >= 10


def test_group_alg1_lmstream_lr2_and_lr1():
    check_run("LR2S", "lmstream", "R(0.5,3)", 45, 4, 45.0, device_ids=[0, 0])
    check_run("LR1S", "lmstream", "U(1.5)", 32, 3, 32.0, device_ids=[0, 0])


def test_group_config_checks():
    import paper_2111_04289_b200 as P
    with pytest.raises(P.LmsError):
        P.Query("CM2S", device_ids=[0, 0], world=2, rank=1)          # one handle drives all devices
    with pytest.raises(P.LmsError):
        P.Query("CM2S", device_ids=[0, 99])
    with P.Query("CM2S", mode="manual", device_ids=[0, 0]) as q:
        with pytest.raises(P.LmsError):
            from paper_2111_04289_b200.dist import RankHandle
            RankHandle(q)                                            # no caller-side protocol


def _multicast_object_possible():
    """Whether this box lets device 0 create a multicast object (CU_DEVICE_ATTRIBUTE_MULTICAST_
    SUPPORTED and cuMulticastCreate through ctypes; a single-GPU container may report the
    attribute but refuse the object)."""
    import ctypes as C
    try:
        cu = C.CDLL("libcuda.so.1")
    except OSError:
        return False
    if cu.cuInit(0) != 0:
        return False
    dev, v = C.c_int(), C.c_int()
    if cu.cuDeviceGet(C.byref(dev), 0) != 0 or cu.cuDeviceGetAttribute(C.byref(v), 132, dev) != 0 or not v.value:
        return False

    class Prop(C.Structure):
        _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t), ("handleTypes", C.c_ulonglong),
                    ("flags", C.c_ulonglong)]
    for ht in (0, 1, 8):
        p = Prop(1, 2 << 20, ht, 0)
        h = C.c_ulonglong()
        if cu.cuMulticastCreate(C.byref(h), C.byref(p)) == 0:
            cu.cuMemRelease(h)
            return True
    return False


def _nvls_active(qname, **cfg):
    import ctypes as C
    import paper_2111_04289_b200 as P
    from paper_2111_04289_b200 import _lib as L
    with P.Query(qname, mode="manual", **cfg) as q:
        a = C.c_int32()
        L.check(L.lms_nvls_active(q.h, C.byref(a)), "lms_nvls_active")
        return a.value


@pytest.mark.parametrize("qname,traffic,secs,bs,G", [
    ("LR2S", "B(1.7)", 45, [3, 7, 1, 10, 4], 2),
    ("LR2S", "R(0.5,2)", 40, [9, 9, 9], 3),
    ("CM1S", "B(0.9)", 75, [10, 10, 3, 20], 2),
    ("CM1T", "U(0.5)", 130, [30, 30, 60], 3),
])
def test_group_nvls_dense_merge(qname, traffic, secs, bs, G):
    """Dense tables (LR2, CM1) merged through NVLS: the close's partial rows are reduced in the
    NVLink switch into every device's replica of one multicast object (multimem.red), owners
    finalize from their replica and zero their keys everywhere (multimem.st).  On a device with
    switch multicast the group handle with LMS_FLAG_NVLS must take that path; without the flag
    (or where no multicast object can be created) the owner push — both against the oracle."""
    from paper_2111_04289_b200 import _lib as L
    fam = qname[:2]
    params = g.CMParams(num_jobs=200) if fam == "CM" else None
    data = stream(fam, traffic, secs, params=params)
    batches, i = [], 0
    for n in bs:
        batches.append(data[i:i + n])
        i += n
    if i < len(data):
        batches.append(data[i:])
    want = oracle_rows(qname, batches)
    assert _nvls_active(qname, device_ids=[0] * G, flags=L.LMS_FLAG_NVLS) == (1 if _multicast_object_possible() else 0)
    assert _nvls_active(qname, device_ids=[0] * G) == 0
    assert _nvls_active("CM2S", device_ids=[0] * G, flags=L.LMS_FLAG_NVLS) == 0   # sparse keys: owner push
    compare_run(qname, product_run(qname, batches, device_ids=[0] * G, flags=L.LMS_FLAG_NVLS), want)
    compare_run(qname, product_run(qname, batches, device_ids=[0] * G), want)
