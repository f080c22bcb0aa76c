"""North-star acceptance at the bench's full size (BASELINE configs[1]): 10 epochs of
the 2-layer GCN over all 8 reddit-shaped SPRING partitions (s = 1, Adam 0.01) on the
B200, against the float64 oracle (oracle/gnn_oracle.py) run on the host cores — the
per-epoch loss within 1e-3 relative and the final test accuracy on the global graph
within 0.5 pt.  The oracle's 8 replicas run in 8 worker processes (one partition
each; the averaging is done in partition order in the parent, as the reference's
model_average).  Output: one JSON line (gpurun_out/fullscale_ten_epochs.json).

    python scripts/fullscale_ten_epochs.py [EPOCHS] [WORKLOAD]   (reddit_gcn | products_sage)

The oracle half alone is frozen into tests/golden/fullscale_<workload>.json by
tests/golden/make_fullscale_fixture.py; tests/test_gpu_fullscale.py runs the B200
half against that fixture on every GPU test run.

products_sage: eight float64 oracle workers over the 1.3 M-row partitions exceed the
196 GB of host RAM on this pool's boxes (a worker died after 47 min); only reddit_gcn
has been run to completion.
"""
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
EPOCHS = 10
WORKLOAD = "reddit_gcn"
SEED, HIDDEN, LR = 7, 256, 0.01


def oracle_shard(prep, i):
    from oracle import gnn_oracle as go, ref
    from benchdata import workloads as W
    p = W.load_part(prep, i)
    rows = p["ext"].size
    local = np.searchsorted(p["ext"], p["edges"].ravel()).astype(np.uint32).reshape(-1, 2)
    off, nb = ref.build_adjacency(rows, local)
    train = np.nonzero((p["owner"] == 1) & (p["role"] == 1))[0].astype(np.int64)
    return go.OracleShard(go.Graph.from_csr(off, nb, rows), p["features"].astype(np.float64),
                          p["labels"].astype(np.int64), train)


def worker(prep, i, init_flat, conn, name):
    from threadpoolctl import threadpool_limits
    threadpool_limits(max(1, (os.cpu_count() or 8) // 8))
    from oracle import gnn_oracle as go
    sh = oracle_shard(prep, i)
    w = _workload(name)
    kind = _kind(w)
    like = go.init_params(kind, w.layers, sh.X.shape[1], HIDDEN, w.classes, seed=SEED)
    rep = go.Replica(kind, go.unflatten(init_flat, like), lr=LR)
    conn.send(len(sh.train_rows))
    while True:
        msg = conn.recv()
        if msg is None:
            break
        rep.params = go.unflatten(msg, like)
        loss = rep.step(sh)
        conn.send((loss, go.flatten(rep.params)))


def _workload(name=None):
    from benchdata import workloads as W
    return W.WORKLOADS[name or WORKLOAD]


def _kind(w):
    from oracle import gnn_oracle as go
    return {"gcn": go.GCN, "sage": go.SAGE, "gin": go.GIN}[w.model]


def load_global(prep):
    from benchdata import workloads as W  # noqa: F401
    X = np.load(os.path.join(prep["dir"], "features.npy"), mmap_mode="r")
    labels = np.load(os.path.join(prep["dir"], "labels.npy"))
    roles = np.load(os.path.join(prep["dir"], "roles.npy"))
    raw = np.fromfile(os.path.join(prep["dir"], "edges.bin"), dtype=np.uint8)
    edges = raw[4:].view(np.uint64).reshape(-1, 2)
    return X, labels, roles, edges


def run_gpu(epochs=EPOCHS, name=None):
    """The B200 half: all partitions through the library (s = 1), then the
    averaged model's test accuracy on the global graph.  Returns a dict."""
    from benchdata import workloads as W
    from paper_2404_02300_b200 import gnn, gnnpart as gp
    w = _workload(name)
    prep = W.prepare(w, lambda *a: None)
    t0 = time.time()
    ctx = gp.Context(0)
    X, labels, roles, edges = load_global(prep)
    shards, counts = [], []
    for i in range(w.partitions):
        p = W.load_part(prep, i, X, labels)
        shards.append(gp.Shard.from_part(p["ext"], p["owner"], p["role"], p["labels"], p["edges"], p["features"], ctx))
        counts.append(int(np.sum((p["owner"] == 1) & (p["role"] == 1))))
    res = gnn.distributed_train(w.model, shards, counts, 1, epochs, w.layers, HIDDEN, w.classes, seed=SEED, lr=LR,
                                ctx=ctx)
    del shards
    # global graph (the full stream, train.cpp:229-238) for the test accuracy
    V = labels.size
    test = np.nonzero(roles == 3)[0]
    gsh = gp.Shard.from_edges(V, edges.astype(np.uint32), np.ascontiguousarray(X, np.float32), ctx)
    m = gnn.GNNModel(w.model, w.layers, w.dim, HIDDEN, w.classes, seed=SEED, ctx=ctx)
    m.set_params(res.params)
    logits, _ = m.forward(gsh, logits=True)
    acc = float(np.mean(np.argmax(logits[test], axis=1) == labels[test]))
    return dict(losses=list(res.losses), test_acc=acc, test_rows=int(test.size), counts=counts,
                seconds=round(time.time() - t0, 1), key=w.key(), meta=prep["meta"])


def run_oracle(epochs=EPOCHS, name=None):
    """The float64 oracle half: one worker process per partition (averaging in
    partition order in the parent, as model_average), then the test accuracy of
    the averaged model on the global graph."""
    from oracle import gnn_oracle as go
    from benchdata import workloads as W
    w = _workload(name)
    prep = W.prepare(w, lambda *a: None)
    X, labels, roles, edges = load_global(prep)
    kind = _kind(w)
    like = go.init_params(kind, w.layers, w.dim, HIDDEN, w.classes, seed=SEED)
    init_flat = go.flatten(like)
    t1 = time.time()
    ctxm = mp.get_context("fork")
    pipes, workers = [], []
    for i in range(w.partitions):
        a, b = ctxm.Pipe()
        pr = ctxm.Process(target=worker, args=(prep, i, init_flat, b, w.name))
        pr.start()
        pipes.append(a)
        workers.append(pr)
    counts = [c.recv() for c in pipes]
    alpha = go.sync_weights(counts)
    shared = init_flat
    losses = []
    for _ in range(epochs):
        for c in pipes:
            c.send(shared)
        out = [c.recv() for c in pipes]
        losses.append(sum(a * o[0] for a, o in zip(alpha, out)))
        flat = np.zeros_like(shared)
        for a, o in zip(alpha, out):
            flat = flat + a * o[1]
        shared = flat
    for c in pipes:
        c.send(None)
    for pr in workers:
        pr.join()
    V = labels.size
    test = np.nonzero(roles == 3)[0]
    G = go.Graph.from_csr(*oracle_global_csr(edges, V), V)
    params = go.unflatten(shared, like)
    fl = go.Replica(kind, params).flags(w.dim)
    H, Zs, _ = go.forward(kind, params, G, np.asarray(X, np.float64), fl)
    acc = float(np.mean(np.argmax(Zs[-1][test], axis=1) == labels[test]))
    return dict(losses=losses, test_acc=acc, test_rows=int(test.size), counts=counts,
                seconds=round(time.time() - t1, 1), key=w.key(), meta=prep["meta"])


def main():
    global EPOCHS, WORKLOAD
    EPOCHS = int(sys.argv[1]) if len(sys.argv) > 1 else EPOCHS
    WORKLOAD = sys.argv[2] if len(sys.argv) > 2 else WORKLOAD
    w = _workload()
    g = run_gpu(EPOCHS)
    o = run_oracle(EPOCHS)
    assert o["counts"] == g["counts"], (o["counts"], g["counts"])
    rel = [abs(a - b) / abs(b) for a, b in zip(g["losses"], o["losses"])]
    line = {"check": f"{w.name} {EPOCHS}-epoch loss and final test accuracy, B200 vs float64 oracle",
            "epochs": EPOCHS, "partitions": w.partitions, "sync_interval": 1, "seed": SEED,
            "loss_gpu": g["losses"], "loss_oracle": o["losses"], "max_rel_loss_err": max(rel),
            "test_acc_gpu": g["test_acc"], "test_acc_oracle": o["test_acc"],
            "acc_diff_pt": 100 * abs(g["test_acc"] - o["test_acc"]), "test_rows": g["test_rows"],
            "pass": bool(max(rel) <= 1e-3 and 100 * abs(g["test_acc"] - o["test_acc"]) <= 0.5),
            "seconds": {"gpu_incl_load": g["seconds"], "oracle_procs": o["seconds"]}}
    print(json.dumps(line), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "fullscale_ten_epochs.json"), "w") as f:
        f.write(json.dumps(line) + "\n")


def oracle_global_csr(edges, V):
    from oracle import ref
    return ref.build_adjacency(V, edges.astype(np.uint32))


if __name__ == "__main__":
    main()
