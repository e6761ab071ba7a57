"""bench.py's N > 1 path end to end: torchrun with 2 ranks (one process per rank) through the
multi-GPU protocol (partial-mode close, owner bucketing, all-to-all, owner merge).  The test box
has one GPU, so both ranks share it and the collectives use gloo with host staging
(LMS_DIST_BACKEND=gloo); on an 8-GPU node the same code runs NCCL on the library streams."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("workload,exchange", [("cm2", "alltoall"), ("lr2", "alltoall"), ("cm2", "p2p"),
                                               ("lr2", "p2p-async"), ("cm2", "device"), ("lr2", "dense"),
                                               ("cm2", "auto")])
def test_torchrun_two_ranks(workload, exchange):
    env = dict(os.environ, LMS_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", workload, "--secondary", "",
           "--e2e-steps", "1", "--no-cpu-baseline", "--exchange", exchange]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["global_batch"] == 2 * 10_000_000
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


@pytest.mark.parametrize("workload", ["cm2", "lr2"])
def test_torchrun_two_ranks_strong_scaling(workload):
    """--scaling strong: 10M records in total per step, each rank's part cut at record boundaries
    by lms_split; the JSON line reports the whole job (global_batch = 10M)."""
    env = dict(os.environ, LMS_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--workload", workload, "--secondary", "",
           "--e2e-steps", "1", "--no-cpu-baseline", "--scaling", "strong"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["config"]["global_batch"] == 10_000_000
