"""bench.py's N > 1 path (the driver's scaling runs launch it under torch.distributed.run, one rank per GPU
over NCCL) exercised on a one-GPU box: two ranks share cuda:0 with host-staged gloo collectives
(SDAS_BENCH_BACKEND=gloo, a test hook).  Weak scaling: world 2 at s seeds per GPU covers the same grid as
world 1 at 2s seeds, so the all-reduced event counts of the timed steps must be equal, and the JSON line
must carry the whole-job figures."""
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


def _line(out):
    return json.loads([ln for ln in out.splitlines() if ln.startswith("{")][-1])


def test_bench_world2_equals_world1():
    common = ["--steps", "2", "--warmup", "3", "--no-cpu-baseline", "--no-flush-leg"]
    env = dict(os.environ, SDAS_BENCH_BACKEND="gloo")
    one = subprocess.run([sys.executable, "bench.py", "--gpus", "1", "--seeds", "32"] + common, cwd=ROOT,
                         capture_output=True, text=True, timeout=900, env=env)
    assert one.returncode == 0, one.stderr[-3000:]
    two = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                          "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
                          "--seeds", "16"] + common, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert two.returncode == 0, two.stderr[-3000:]
    a, b = _line(one.stdout), _line(two.stdout)
    assert b["n_gpus"] == 2 and a["n_gpus"] == 1
    assert b["config"]["replicas_per_step"] == a["config"]["replicas_per_step"] == 64 * 8 * 32
    assert b["events_per_step"] == a["events_per_step"]                 # all-reduced cells == one-rank cells
    for k in ("value", "ms_per_step"):
        assert b[k] > 0
    assert b["e2e"]["value"] > 0 and b["gpu_launches"] == 8
    assert len([ln for ln in two.stdout.splitlines() if ln.startswith("{")]) == 1   # rank 0 prints alone
