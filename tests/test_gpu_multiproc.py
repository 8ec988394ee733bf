"""The N > 1 bench path end to end on a one-GPU box: two torchrun ranks share
the device over gloo (GP_DIST_BACKEND=gloo) — sizes-first allgather, the
concurrent peer decode, max-over-ranks timing, one JSON line from rank 0.
A functional check only: numbers from such a run are not bench values."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("config", ["c2", "c4"])
def test_two_rank_bench_runs(config):
    env = dict(os.environ, GP_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config",
           config, "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    p = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "dp2"
    assert line["e2e"]["output_check"] is True
