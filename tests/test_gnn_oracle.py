"""Pins the GNN restatement (oracle/gnn_oracle.py) to the compiled reference
(oracle/_ref = /root/reference/proj/src/*.cpp unmodified):

* its aggregation primitive with mean-with-self normalisation equals
  sgc_propagate (train.cpp:49-65);
* its last-layer loss / dlogits / weight gradient equal softmax_loss /
  softmax_gradient (train.cpp:74-94), its averaging equals model_average
  (:154-172), its micro-F1 equals evaluate_micro_f1 (:174-198);
* its whole partition-parallel loop, run with the SGC kind (one layer,
  D~^-1 (A+I) h W^T + b, zero init, SGD, full batch), reproduces the
  reference's own distributed_train (:289-340) with prop_hops = 1 and a batch
  larger than every train set, on real artifacts the reference partitioned;
* its backward matches central differences of its own forward for every layer
  kind / layout."""
import numpy as np
import pytest

from conftest import make_artifact, make_dataset
from oracle import gnn_oracle as go
from oracle import ref

FULL_BATCH = 2 ** 31


def small_graph(rows=40, edges=150, seed=0):
    rng = np.random.default_rng(seed)
    pairs = rng.integers(0, rows, size=(edges, 2))
    pairs[::9, 1] = pairs[::9, 0]
    off, nb = ref.build_adjacency(rows, pairs)
    return go.Graph.from_csr(off, nb, rows), off, nb


def test_aggregate_is_sgc_propagate():
    G, off, nb = small_graph()
    x = np.random.default_rng(1).normal(size=(40, 6))
    np.testing.assert_allclose(G.aggregate(G.aggregate(x, "sgc", True), "sgc", True),
                               ref.sgc_propagate(off, nb, x, 2), rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("kind,in_dim,hidden,classes,layers", [
    (go.GCN, 5, 7, 3, 2), (go.GCN, 9, 4, 3, 2), (go.SAGE, 3, 6, 4, 2), (go.SAGE, 8, 5, 3, 3),
    (go.GIN, 4, 6, 3, 2), (go.SGC, 6, 5, 4, 1), (go.SGC, 3, 5, 4, 2)])
def test_oracle_gradcheck(kind, in_dim, hidden, classes, layers):
    G, _, _ = small_graph(seed=kind)
    rng = np.random.default_rng(7)
    X = rng.normal(size=(40, in_dim))
    labels = rng.integers(0, classes, 40)
    sh = go.OracleShard(G, X, labels, np.arange(0, 40, 2))
    params = go.init_params(kind, layers, in_dim, hidden, classes, seed=3)
    if kind == go.SGC:  # zero init has dead ReLUs; check the gradient at a random point
        params = go.unflatten(rng.normal(size=go.flatten(params).size) * 0.5, params)
    rep = go.Replica(kind, params)
    loss, H, Zs, grads = rep.forward_backward(sh)
    flat = go.flatten(params)
    g = go.flatten(grads)
    idx = rng.choice(flat.size, size=min(40, flat.size), replace=False)
    for i in idx:
        for sgn in (1, -1):
            pass
        fp = flat.copy(); fp[i] += 1e-6
        fm = flat.copy(); fm[i] -= 1e-6
        rep.params = go.unflatten(fp, params); lp = rep.forward_backward(sh)[0]
        rep.params = go.unflatten(fm, params); lm = rep.forward_backward(sh)[0]
        num = (lp - lm) / 2e-6
        assert abs(num - g[i]) <= 1e-6 + 1e-4 * abs(g[i]), (i, num, g[i])


def test_sync_weights_restatement_matches_reference():
    for counts in ([1, 3], [5, 0], [7, 11, 13]):
        assert np.array_equal(np.array(go.sync_weights(counts)), ref.sync_weights(counts))


def test_last_layer_loss_and_gradient_match_reference():
    # SGC-kind layer: Z = (A~ X) W^T + b, so loss / dW / db are the reference's
    # softmax_loss / softmax_gradient over the train rows of the propagated features
    G, off, nb = small_graph(rows=60, edges=260, seed=4)
    rng = np.random.default_rng(5)
    X = rng.normal(size=(60, 7))
    labels = rng.integers(0, 5, 60)
    labels[0] = 4
    train = np.sort(rng.choice(60, 33, replace=False))
    W = rng.normal(size=(5, 7)) * 0.4
    b = rng.normal(size=5) * 0.2
    rep = go.Replica(go.SGC, [[W, b]], optimizer=go.SGD)
    loss, H, Zs, grads = rep.forward_backward(go.OracleShard(G, X, labels, train))
    xp = ref.sgc_propagate(off, nb, X, 1)[train]
    y = labels[train]
    assert abs(loss - ref.softmax_loss(W.T, b, xp, y)) <= 1e-13 * abs(loss)
    gW, gb = ref.softmax_gradient(W.T, b, xp, y)
    np.testing.assert_allclose(grads[0][0], gW.T, rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(grads[0][1], gb, rtol=1e-11, atol=1e-14)
    # dlogits: softmax rows minus one-hot over the train rows / n_train (train.cpp:86-94)
    _, dZ = go.loss_and_dlogits(Zs[-1], labels, train)
    assert np.all(dZ[np.setdiff1d(np.arange(60), train)] == 0)
    np.testing.assert_allclose(xp.T @ dZ[train], gW, rtol=1e-11, atol=1e-14)


def test_model_average_matches_reference():
    rng = np.random.default_rng(8)
    for counts in ([1, 3], [5, 0], [7, 11, 13, 2]):
        reps = [[[rng.normal(size=(4, 6)), rng.normal(size=4)]] for _ in counts]
        avg = go.model_average(reps, counts)
        W, b = ref.model_average(np.stack([r[0][0].T for r in reps]), np.stack([r[0][1] for r in reps]), counts)
        assert np.array_equal(avg[0][0], W.T) and np.array_equal(avg[0][1], b)


def test_micro_f1_matches_reference():
    rng = np.random.default_rng(9)
    x = rng.normal(size=(80, 5))
    W = rng.normal(size=(5, 6))
    b = np.zeros(6)
    b[2] = 10.0  # ties and dominance exercise the first-max rule
    labels = rng.integers(0, 6, 80)
    for mask in (np.arange(80), np.arange(0, 80, 3)):
        assert go.micro_f1(x @ W + b, labels, mask) == ref.evaluate_micro_f1(W, b, x, labels, mask)
    Wt = np.zeros((5, 6))  # all logits equal: first index wins
    assert go.micro_f1(x @ Wt, labels, np.arange(80)) == ref.evaluate_micro_f1(Wt, b * 0, x, labels, np.arange(80))


@pytest.mark.parametrize("p,sync,epochs", [(2, 1, 4), (2, 3, 7), (4, 2, 5)])
def test_sgc_kind_distributed_train_matches_reference(tmp_path, p, sync, epochs):
    ds = make_dataset(tmp_path, scale=10, edges=4000, dim=12, classes=5, seed=p + sync)
    art = make_artifact(ds, p=p)
    td = ref.TrainingData(art)
    lr = 0.5
    rr = td.distributed_train(1, sync, epochs=epochs, lr=lr, batch=FULL_BATCH, prop_hops=1, seed=3)
    shards = [go.shard_from_ref(td.shard(s)) for s in range(p)]
    glob = go.shard_from_ref(td.shard(-1))
    classes = int(glob.labels.max()) + 1
    res = go.distributed_train(go.SGC, shards, sync, epochs, 1, 0, classes, seed=0, optimizer=go.SGD, lr=lr,
                               global_shard=glob)
    W, b = res["params"][0]
    np.testing.assert_allclose(W.T, rr["W"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(b, rr["b"], rtol=1e-9, atol=1e-12)
    assert res["averaging_ops"] == rr["averaging_ops"]
    assert [h[:2] for h in res["history"]] == [tuple(h[:2]) for h in rr["history"]]
    np.testing.assert_allclose(np.array([h[2:] for h in res["history"]]), np.array([h[2:] for h in rr["history"]]),
                               atol=1e-12)
