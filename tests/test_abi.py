"""C-ABI contract tests (CPU): the library loads, exports every declared symbol, and its pure
cost-model functions agree with the SPEC worked examples and with the oracle."""
import ctypes as C
import math
import os
import random
import re

import pytest

from oracle import planner as OP
from oracle import regression as OG
from oracle import sizer as OZ

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2111_04289_b200 import build
    build.build()
    from paper_2111_04289_b200 import _lib
    return _lib


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "lmstream.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lms_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(L):
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L._lib, s), s
    assert set(syms) == set(L.EXPORTED)


def test_abi_version_and_struct_sizes(L, tmp_path):
    assert L.lms_abi_version() == L.LMS_ABI_VERSION == 3
    assert C.sizeof(L.lms_agg_row) == 72
    assert C.sizeof(L.lms_lr1_row) == 32
    # the ctypes mirrors match the C compiler's layout of include/lmstream.h
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include "lmstream.h"\nint main(void){printf("%zu %zu %zu %zu %zu\\n",'
                   ' sizeof(lms_config), sizeof(lms_batch_record), sizeof(lms_agg_row), sizeof(lms_lr1_row),'
                   ' sizeof(lms_dag)); return 0;}\n')
    exe = tmp_path / "sz"
    import subprocess
    subprocess.run(["gcc", "-std=c99", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got == [C.sizeof(L.lms_config), C.sizeof(L.lms_batch_record), C.sizeof(L.lms_agg_row),
                   C.sizeof(L.lms_lr1_row), C.sizeof(L.lms_dag)]


def test_config_defaults_and_validation(L):
    cfg = L.lms_config()
    assert L.lms_config_init(C.byref(cfg), L.LMS_CM2S) == 0
    assert cfg.struct_size == C.sizeof(L.lms_config)
    assert cfg.inf_pt_bytes == 150e3 and cfg.base_trans_cost == 0.1 and cfg.num_cores == 12
    assert L.lms_config_init(C.byref(cfg), 99) == L.LMS_EINVAL
    h = C.c_void_p()
    bad = L.lms_config()
    L.lms_config_init(C.byref(bad), L.LMS_LR2S)
    bad.struct_size = 4
    assert L.lms_query_create(C.byref(bad), C.byref(h)) == L.LMS_EINVAL
    L.lms_config_init(C.byref(bad), L.LMS_LR2S)
    bad.slide_s, bad.range_s = 7, 30                      # S must divide R
    st = L.lms_query_create(C.byref(bad), C.byref(h))
    assert st in (L.LMS_EINVAL, L.LMS_ECUDA)
    assert L.lms_last_error()


def test_create_without_gpu_reports_ecuda(L):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    cfg = L.lms_config()
    L.lms_config_init(C.byref(cfg), L.LMS_LR2S)
    h = C.c_void_p()
    assert L.lms_query_create(C.byref(cfg), C.byref(h)) == L.LMS_ECUDA
    assert b"CUDA" in L.lms_last_error() or b"device" in L.lms_last_error()


def _d(x):
    return C.c_double(x)


def test_cost_models_spec_examples(L):
    out = C.c_double()
    for fn, args, want in ((L.lms_cpu_cost, (1.0, 15e3, 150e3), 0.1), (L.lms_cpu_cost, (0.8, 1500e3, 150e3), 8.0),
                           (L.lms_gpu_cost, (1.0, 15e3, 150e3), 10.0), (L.lms_gpu_cost, (0.8, 1500e3, 150e3), 0.08),
                           (L.lms_trans_cost, (0.1, 150e3, 150e3), 0.1), (L.lms_trans_cost, (0.1, 1.5e6, 150e3), 1.0)):
        assert fn(*args, C.byref(out)) == 0
        assert out.value == pytest.approx(want)
    assert L.lms_cpu_cost(1.0, 0.0, 1.0, C.byref(out)) == L.LMS_EINVAL
    for k in range(8):
        assert L.lms_base_cost(k, C.byref(out)) == 0
        assert out.value == OP.BASE_COST[k]
    assert L.lms_base_cost(8, C.byref(out)) == L.LMS_EINVAL


def _dag_arrays(dag):
    kinds = (C.c_uint8 * len(dag))(*[k for k, _ in dag])
    offs, preds = [0], []
    for _, p in dag:
        preds += p
        offs.append(len(preds))
    o = (C.c_int32 * len(offs))(*offs)
    p = (C.c_int32 * max(1, len(preds)))(*preds)
    return kinds, o, p


def test_map_device_matches_oracle_alg2(L):
    rng = random.Random(1)
    for name, dag in OP.DAGS.items():
        kinds, o, p = _dag_arrays(dag)
        d = L.lms_dag(len(dag), kinds, o, p)
        out = (C.c_uint8 * len(dag))()
        for _ in range(300):
            part, inf = rng.uniform(1e3, 1e7), rng.uniform(1e3, 1e7)
            assert L.lms_map_device(C.byref(d), part, inf, 0.1, out) == 0
            assert list(out) == OP.map_device(dag, part, inf), (name, part, inf)
    cyc = [(OP.SCAN, [1]), (OP.FILTER, [0])]
    kinds, o, p = _dag_arrays(cyc)
    d = L.lms_dag(2, kinds, o, p)
    out = (C.c_uint8 * 2)()
    assert L.lms_map_device(C.byref(d), 1e5, 1e5, 0.1, out) == L.LMS_EPLAN


def test_query_dag_catalog(L):
    d = L.lms_dag()
    for kind, name in ((0, "LR1"), (2, "LR2"), (3, "CM1"), (5, "CM2")):
        assert L.lms_query_dag(kind, C.byref(d)) == 0
        dag = [(d.op_kind[i], [d.preds[j] for j in range(d.pred_off[i], d.pred_off[i + 1])]) for i in range(d.n)]
        assert dag == [(k, list(p)) for k, p in OP.DAGS[name]]


def test_est_max_lat_and_admission_match_oracle(L):
    out = C.c_double()
    buff = (C.c_double * 2)(1.0, 2.0)
    by = (C.c_uint64 * 2)(2_000_000, 2_000_000)
    assert L.lms_est_max_lat(buff, by, 2, 2e6, C.byref(out)) == 0 and out.value == pytest.approx(4.0)
    assert L.lms_est_max_lat(buff, by, 0, 2e6, C.byref(out)) == L.LMS_EINVAL
    rng = random.Random(9)
    adm, est, reason = C.c_int32(), C.c_double(), C.c_int32()
    for trial in range(2000):
        n = rng.randrange(0, 6)
        now = rng.uniform(0, 100)
        ds = sorted((now - rng.uniform(0, 8), rng.randrange(1, 10 ** 7)) for _ in range(n))
        thp = rng.choice([0.0, rng.uniform(1e5, 1e8)])
        hist = [rng.uniform(0.1, 10) for _ in range(rng.randrange(0, 4))]
        mode = rng.choice(["lmstream", "deadline"])
        slide = rng.choice([0.0, 5.0, 10.0])
        dl = rng.choice([0.0, 1.0, 5.0])
        ing = (C.c_double * max(1, n))(*[x for x, _ in ds])
        byt = (C.c_uint64 * max(1, n))(*[b for _, b in ds])
        hh = (C.c_double * max(1, len(hist)))(*hist)
        assert L.lms_admit_decision(0 if mode == "lmstream" else 1, slide, dl, now, ing, byt, n, thp, hh,
                                    len(hist), C.byref(adm), C.byref(est), C.byref(reason)) == 0
        dsets = [OZ.Dataset(i, x, b) for i, (x, b) in enumerate(ds)]
        o = OZ.construct_micro_batch([], dsets, now, mode=mode, slide_s=slide, deadline_s=dl,
                                     avg_thput_prev=thp if thp > 0 else None, max_lat_history=hist)
        assert bool(adm.value) == o.admitted, trial
        if o.est_max_lat is not None:
            assert est.value == pytest.approx(o.est_max_lat, rel=1e-12)


def test_regression_matches_oracle(L):
    rng = random.Random(3)
    b0, b1, b2 = C.c_double(), C.c_double(), C.c_double()
    for _ in range(50):
        n = rng.randrange(3, 40)
        th = [rng.uniform(1e6, 1e9) for _ in range(n)]
        la = [rng.uniform(0.01, 10) for _ in range(n)]
        ip = [rng.uniform(1e3, 1e7) for _ in range(n)]
        A = (C.c_double * n)
        assert L.lms_infpt_fit(A(*th), A(*la), A(*ip), n, C.byref(b0), C.byref(b1), C.byref(b2)) == 0
        want = OG.fit(zip(th, la, ip))
        for got, w in zip((b0.value, b1.value, b2.value), want):
            assert got == pytest.approx(w, rel=1e-6, abs=1e-6 * max(abs(x) for x in want))
    A = (C.c_double * 2)
    assert L.lms_infpt_fit(A(1, 2), A(1, 2), A(1, 2), 2, C.byref(b0), C.byref(b1), C.byref(b2)) == L.LMS_EHISTORY
    out = C.c_double()
    assert L.lms_infpt_predict(-5e3, 0, 0, 1, 1, C.byref(out)) == 0 and out.value == 1024.0


def test_percentile(L):
    out = C.c_double()
    v = (C.c_double * 100)(*range(1, 101))
    assert L.lms_percentile(v, 100, 99, C.byref(out)) == 0 and out.value == 99
    v = (C.c_double * 10)(*range(1, 11))
    assert L.lms_percentile(v, 10, 99, C.byref(out)) == 0 and out.value == 10
    assert L.lms_percentile(v, 0, 99, C.byref(out)) == L.LMS_EINVAL
    assert not math.isnan(out.value)
