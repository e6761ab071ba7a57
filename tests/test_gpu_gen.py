"""The CUDA generator (lmsgen/gen.cu) reproduces the Python generator byte for byte."""
import pytest

import lmsgen as g

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("family,params", [("LR", g.LRParams()), ("LR", g.LRParams(num_xways=16, num_vehicles=77)),
                                            ("CM", g.CMParams()), ("CM", g.CMParams(num_jobs=50, sel_ppm=100000))])
def test_cuda_generator_matches_python(family, params):
    from lmsgen import cuda as gc
    for t, count in ((0, 1), (7, 3000), (123456, 777)):
        buf, n = gc.second_tensor(family, t, count, params=params)
        got = bytes(buf[:n].cpu().numpy())
        want = g.second_bytes(family, t, count, params=params)
        assert got == want


def test_cuda_generator_sampled_at_full_rate():
    from lmsgen import cuda as gc
    buf, n = gc.second_tensor("CM", 3, 10_000_000)
    data = bytes(buf[:n].cpu().numpy())
    lines = data.split(b"\n")[:-1]
    assert len(lines) == 10_000_000
    for i in (0, 1, 4_999_999, 9_999_999):
        assert lines[i] + b"\n" == g.cm_record(g.SEED, 3, i)
    buf, n = gc.second_tensor("LR", 3, 10_000_000)
    assert n == 700_000_000
    for i in (0, 5_000_001, 9_999_999):
        assert bytes(buf[70 * i:70 * i + 70].cpu().numpy()) == g.lr_record(g.SEED, 3, i)
