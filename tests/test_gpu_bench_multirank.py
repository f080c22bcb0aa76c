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


def test_bench_self_launches_n_ranks():
    """`python bench.py --gpus 2` with no launcher re-executes itself as 2 ranks
    (torch.distributed.run); on a one-GPU box the ranks share the device with
    host collectives, and the line says so."""
    env = dict(os.environ, CATGNN_WORKLOAD="tiny_gcn")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3",
                          "--no-cpu-baseline"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["config"]["partitions_per_gpu"] == 2
    import torch
    if torch.cuda.device_count() < 2:
        assert d["config"]["shared_devices"] is True and "gloo" in d["config"]["collectives"]


@pytest.mark.parametrize("graph,lanes,sync", [(1, 1, 1), (0, 1, 1), (1, 2, 1), (1, 1, 4)])
def test_bench_single_rank_contract(graph, lanes, sync):
    """The one-GPU bench line (driver contract): graph-replayed and eager steps,
    shard lanes; every key the driver and the judge read is present and sane."""
    env = dict(os.environ, CATGNN_WORKLOAD="tiny_gcn")
    cmd = [sys.executable, "bench.py", "--steps", "4", "--warmup", "3", "--graph", str(graph),
           "--lanes", str(lanes), "--sync", str(sync)]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks", "step_breakdown"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["value"] > 0 and d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] in ("hbm", "l2") and r["achieved"] > 0 and r["peak"] > 0 and r["unit"] == "GB/s"
    assert 0 < r["frac"] <= 1.2 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert (e["graph"] is not None) == (bool(graph) and sync == 1)
    assert "graph capture failed" not in out.stderr
    assert any(k.startswith("K2 agg") for k in d["step_breakdown"])


def test_bench_reference_arm_line():
    env = dict(os.environ, CATGNN_WORKLOAD="tiny_gcn")
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "2", "--warmup", "1"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
