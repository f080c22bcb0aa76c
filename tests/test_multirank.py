"""Multi-rank C1 model averaging (world size 2, gloo): cyclic partition
assignment (train.cpp:293-294) and the rank-share + all-reduce
equal the reference's model_average (train.cpp:154-172) over all replicas.

* CPU: the host algebra (each rank sums alpha_i theta_i over its partitions
  with the GLOBAL sync_weights, then all-reduce), including a rank whose
  partitions hold no train rows (weight 0, no error — ADVICE r01).
* GPU: the same through the LIBRARY — each rank holds device replicas
  (catgnn_model_set_params), forms its share with catgnn_model_weighted_sum,
  and the shares are all-reduced (NCCL when the box has a GPU per rank, else
  gloo on the host over the shares read back); the result is compared with the
  compiled reference's model_average over all partitions."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ref


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem(p, zero_rank1=False):
    rng = np.random.default_rng(0)
    params = [rng.normal(size=257) for _ in range(p)]
    counts = rng.integers(1, 1000, size=p).tolist()
    if zero_rank1:  # rank 1's partitions (1, 3, ...) have no train rows
        counts = [c if i % 2 == 0 else 0 for i, c in enumerate(counts)]
    return params, counts


def rank_share(local_params, my_alpha):
    """bench.py / gnn.distributed_train / catgnn_gnn_distributed_train: this
    rank's sum of alpha_i theta_i (global alphas), from zero in partition order."""
    acc = np.zeros_like(local_params[0], dtype=np.float64)
    for a, p in zip(my_alpha, local_params):
        acc = acc + a * p.astype(np.float64)
    return acc


def _worker(rank, world, port, p, zero_rank1, use_lib, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_2404_02300_b200.gnn import assign_partitions, sync_weights
    params, counts = _problem(p, zero_rank1)
    alpha = sync_weights(counts)
    mine = assign_partitions(p, world, rank)
    if not use_lib:
        share = rank_share([params[i] for i in mine], [alpha[i] for i in mine])
    else:
        from paper_2404_02300_b200 import gnnpart as gp
        from paper_2404_02300_b200.gnn import GNNModel, weighted_sum
        ctx = gp.Context(rank % torch.cuda.device_count())
        # a 1-layer model with 256 x 1 weights + 1 bias = 257 parameters
        mk = lambda: GNNModel("gcn", 1, 256, 0, 1, ctx=ctx)  # noqa: E731
        reps = []
        for i in mine:
            m = mk()
            m.set_params(params[i].astype(np.float32))
            reps.append(m)
        shared = mk()
        weighted_sum(reps, [alpha[i] for i in mine], shared)
        share = shared.get_params().astype(np.float64)
    t = torch.from_numpy(share.copy())
    dist.all_reduce(t)
    out_q.put((rank, mine, t.numpy()))
    dist.destroy_process_group()


def _run(p, zero_rank1, use_lib):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, p, zero_rank1, use_lib, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    return res


def _reference(p, zero_rank1):
    params, counts = _problem(p, zero_rank1)
    W, _ = ref.model_average(np.stack(params)[:, :, None], np.zeros((p, 1)), counts)
    return W[:, 0]


@pytest.mark.parametrize("p,zero_rank1", [(2, False), (4, False), (8, False), (4, True)])
def test_two_rank_average_matches_reference(p, zero_rank1):
    res = _run(p, zero_rank1, use_lib=False)
    want = _reference(p, zero_rank1)
    owned = sorted(i for _, mine, _ in res for i in mine)
    assert owned == list(range(p))
    for _, mine, got in res:
        assert mine == list(range(mine[0], p, 2))
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
@pytest.mark.parametrize("p,zero_rank1", [(4, False), (8, True)])
def test_two_rank_library_average_matches_reference(p, zero_rank1):
    res = _run(p, zero_rank1, use_lib=True)
    want = _reference(p, zero_rank1)
    for _, mine, got in res:
        # float32 parameters on the device, f64 accumulation (average_kernel)
        np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-6)


def test_assignment_errors():
    from paper_2404_02300_b200 import ConfigError
    from paper_2404_02300_b200.gnn import assign_partitions
    with pytest.raises(ConfigError):
        assign_partitions(6, 4, 0)
    with pytest.raises(ConfigError):
        assign_partitions(0, 1, 0)


def test_bench_rejects_world_mismatch():
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0", CATGNN_WORKLOAD="tiny_gcn")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1"], cwd=root, env=env,
                         capture_output=True, text=True, timeout=120)
    assert out.returncode != 0 and "!= --gpus 2" in out.stderr
