"""Diagnostic: per-intermediate relative errors of one GCN step vs the oracle."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from oracle import gnn_oracle as go, ref
from paper_2404_02300_b200 import gnnpart as gp, synth
from paper_2404_02300_b200.gnn import GNNModel

def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / max(np.linalg.norm(b), 1e-30))

e, n, _ = synth.rmat_edges(11, 12000, seed=4)
hub = np.stack([np.zeros(1500, np.uint64), np.arange(1, 1501, dtype=np.uint64) % n], 1)
pairs = np.concatenate([e, hub[hub[:, 1] != 0]]).astype(np.uint32)
off, nb = ref.build_adjacency(n, pairs)
G = go.Graph.from_csr(off, nb, n)
for kind, in_dim, hidden, classes in [("gcn", 602, 64, 41), ("gcn", 8, 32, 5)]:
    rng = np.random.default_rng(1)
    X = rng.normal(size=(n, in_dim)).astype(np.float32)
    labels = rng.integers(0, classes, n).astype(np.int32)
    train = np.sort(rng.choice(n, size=n // 2, replace=False)).astype(np.uint32)
    s = gp.Shard.from_edges(n, pairs, X); s.set_labels(labels, train)
    m = GNNModel(kind, 2, in_dim, hidden, classes, seed=5)
    p = m.get_params().astype(np.float64)
    loss = m.forward_backward(s)
    init = go.init_params(go.GCN, 2, in_dim, hidden, classes, seed=5)
    params = go.unflatten(p, init)
    o = go.OracleShard(G, X.astype(np.float64), labels, train.astype(np.int64))
    fl = [in_dim < hidden, hidden < classes]
    H, Zs, aux = go.forward(go.GCN, params, G, o.X, fl)
    L, dZ1 = go.loss_and_dlogits(Zs[-1], labels, train)
    W1 = params[1][0]
    dinv = 1 / np.sqrt(1 + G.deg)
    dA1 = dZ1 @ W1
    dh0 = G.aggregate(dA1, "gcn", True, pre=dinv)
    dZ0 = dh0 * (Zs[0] > 0)
    grads = go.backward(go.GCN, params, G, H, Zs, aux, dZ1, fl)
    g = m.unflatten(m.get_grads())
    print(kind, in_dim, "loss", loss, L)
    print(" H0", rel(m.export(0, 0, n), H[1]), " Z1", rel(m.export(1, 0, n), H[2]))
    print(" dZ1", rel(m.export(1, 2, n), dZ1), " dZ0", rel(m.export(0, 2, n), dZ0))
    for l in range(2):
        print(" layer", l, "dW", rel(g[l][0], grads[l][0]), "db", rel(g[l][1], grads[l][1]))
    gw = g[0][0]; rw = grads[0][0]
    rowerr = np.linalg.norm(gw - rw, axis=1) / np.linalg.norm(rw, axis=1)
    print(" dW0 per-row err (max/median):", rowerr.max(), np.median(rowerr), "argmax", rowerr.argmax())
    colerr = np.linalg.norm(gw - rw, axis=0) / np.linalg.norm(rw, axis=0)
    print(" dW0 per-col err (max/median):", colerr.max(), np.median(colerr), "argmax", colerr.argmax())
    # relu mask flips
    gz = m.export(0, 0, n)
    print(" H0 mask flips:", int(np.sum((gz > 0) != (H[1] > 0))), "of", gz.size)
