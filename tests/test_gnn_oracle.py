"""Pins the GNN restatement (oracle/gnn_oracle.py) where the reference allows:
its aggregation primitive with mean-with-self normalisation equals the
reference's sgc_propagate, and its backward matches central differences of its
own forward for every layer kind / layout."""
import numpy as np
import pytest

from oracle import gnn_oracle as go
from oracle import ref


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
    (go.GIN, 4, 6, 3, 2)])
def test_oracle_gradcheck(kind, in_dim, hidden, classes, layers):
    G, _, _ = small_graph(seed=kind)
    rng = np.random.default_rng(7)
    X = rng.normal(size=(40, in_dim))
    labels = rng.integers(0, classes, 40)
    sh = go.OracleShard(G, X, labels, np.arange(0, 40, 2))
    params = go.init_params(kind, layers, in_dim, hidden, classes, seed=3)
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
