"""Multi-rank host logic of the C1 model-averaging step on CPU (gloo, world
size 2): cyclic partition assignment (train.cpp:293-294) and the
alpha-prescaled all-reduce equal the reference's model_average
(train.cpp:154-172) over all replicas."""
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


def rank_average(local_params, local_counts, my_alpha, allreduce):
    """Same algebra as bench.py / gnn.distributed_train on the device:
    weighted mean of the rank's replicas, scaled by the rank's alpha share,
    summed over ranks."""
    c = np.asarray(local_counts, np.float64)
    if len(local_params) == 1:
        acc = local_params[0].astype(np.float64)
    else:
        acc = sum((ci / c.sum()) * p.astype(np.float64) for ci, p in zip(c, local_params))
    acc = acc * float(sum(my_alpha))
    return allreduce(acc)


def _worker(rank, world, port, p, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import torch
    from paper_2404_02300_b200.gnn import assign_partitions, sync_weights
    rng = np.random.default_rng(0)
    params = [rng.normal(size=257) for _ in range(p)]
    counts = rng.integers(1, 1000, size=p).tolist()
    alpha = sync_weights(counts)
    mine = assign_partitions(p, world, rank)

    def allreduce(a):
        t = torch.from_numpy(a.copy())
        dist.all_reduce(t)
        return t.numpy()

    got = rank_average([params[i] for i in mine], [counts[i] for i in mine], [alpha[i] for i in mine], allreduce)
    out_q.put((rank, mine, got))
    dist.destroy_process_group()


@pytest.mark.parametrize("p", [2, 4, 8])
def test_two_rank_average_matches_reference(p):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, p, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    rng = np.random.default_rng(0)
    params = [rng.normal(size=257) for _ in range(p)]
    counts = rng.integers(1, 1000, size=p).tolist()
    W, _ = ref.model_average(np.stack(params)[:, :, None], np.zeros((p, 1)), counts)
    owned = sorted(i for _, mine, _ in res for i in mine)
    assert owned == list(range(p))
    for _, mine, got in res:
        assert mine == list(range(mine[0], p, 2))
        np.testing.assert_allclose(got, W[:, 0], rtol=1e-12, atol=1e-12)


def test_assignment_errors():
    from paper_2404_02300_b200 import ConfigError
    from paper_2404_02300_b200.gnn import assign_partitions
    with pytest.raises(ConfigError):
        assign_partitions(6, 4, 0)
    with pytest.raises(ConfigError):
        assign_partitions(0, 1, 0)
