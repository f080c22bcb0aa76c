"""bench.py's multi-rank flow (torchrun, one process per GPU, cyclic partition
assignment, barriers, alpha-prescaled all-reduce of the averaged model, max-over-
ranks timing) on a single-GPU box: ranks share the device and the all-reduce runs
through gloo on the host (CATGNN_BENCH_HOST_COLLECTIVES=1) instead of NCCL."""
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


def test_bench_two_ranks_host_collectives():
    env = dict(os.environ, CATGNN_BENCH_HOST_COLLECTIVES="1", CATGNN_WORKLOAD="tiny_gcn")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 prints the one JSON line
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["workload"] == "tiny_gcn" and d["gpu_launches"] > 0
