"""TEST INFRASTRUCTURE ONLY — float64 CPU restatement of the north-star GNN
layers (GCN-norm / SAGE-mean / GIN-sum) trained full-batch per partition with
alpha-weighted model averaging.

PARITY UNPINNED BY THE REFERENCE: /root/reference trains only SGC
(proj/src/train.cpp) and has no GCN/SAGE/GIN, so this module restates the
layers under the reference's conventions:
  * CSR and degrees are the LOCAL build_adjacency multiset (train.cpp:30-47,
    :60): duplicates count, a self-loop appears once;
  * loss = mean cross-entropy over the shard's train rows (owner && train,
    train.cpp:266), epoch loss = sum_i alpha_i loss_i;
  * model averaging = sync_weights + model_average over every parameter
    tensor (train.cpp:139-172), chunks of min(s, remaining) local iterations
    (train.cpp:315-323); optimizer state is per replica and not averaged;
  * micro-F1 = pooled TP/(TP+miss) with first-index argmax (train.cpp:174-198).
Pinned to the compiled reference (tests/test_gnn_oracle.py): with
mean-with-self normalisation `aggregate` IS sgc_propagate; the SGC kind (one
layer, D~^-1 (A+I) h W^T + b, zero init, SGD, full batch) reproduces the
reference's own distributed_train (prop_hops = 1, batch >= every train set);
loss / dlogits / dW against softmax_loss / softmax_gradient, `model_average`
against model_average and `micro_f1` against evaluate_micro_f1.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List

import numpy as np
import scipy.sparse as sp

from paper_2404_02300_b200.synth import mix64, seed_for  # common.hpp:27-39 restated

GCN, SAGE, GIN, SGC = 1, 2, 3, 4
SGD, ADAM = 0, 1


def csr_matrix(offsets, neighbors, rows):
    """Multiset adjacency of a LocalAdjacency (entries = multiplicities)."""
    offsets = np.asarray(offsets, np.int64)
    data = np.ones(int(offsets[-1]), np.float64)
    A = sp.csr_matrix((data, np.asarray(neighbors, np.int64), offsets), shape=(rows, rows))
    A.sum_duplicates()
    return A


@dataclass
class Graph:
    A: sp.csr_matrix
    deg: np.ndarray

    @classmethod
    def from_csr(cls, offsets, neighbors, rows):
        off = np.asarray(offsets, np.int64)
        return cls(csr_matrix(off, neighbors, rows), np.diff(off).astype(np.float64))

    def aggregate(self, X, norm, self_term, pre=None):
        """post * (self*pre*X + A (pre*X)) — the K2 primitive."""
        Y = X if pre is None else X * pre[:, None]
        out = self.A @ Y
        if self_term:
            out = out + Y
        return out * self.post(norm)[:, None]

    def post(self, norm):
        d = self.deg
        if norm == "sgc":
            return 1.0 / (1.0 + d)
        if norm == "gcn":
            return 1.0 / np.sqrt(1.0 + d)
        if norm == "mean":
            return np.where(d > 0, 1.0 / np.maximum(d, 1), 0.0)
        return np.ones_like(d)


def layer_dims(kind, layers, in_dim, hidden, classes):
    out = []
    for l in range(layers):
        d_in = in_dim if l == 0 else hidden
        d_out = classes if l + 1 == layers else hidden
        agg_first = d_in <= d_out if kind == SAGE else d_in < d_out
        if kind == SAGE:
            shape = (d_out, 2 * d_in) if agg_first else (2 * d_out, d_in)
        else:
            shape = (d_out, d_in)
        out.append((d_in, d_out, agg_first, shape))
    return out


def init_params(kind, layers, in_dim, hidden, classes, seed):
    """Glorot-uniform from splitmix64(seed_for(seed, layer) + i), biases zero;
    the SGC kind is zero-initialised like the reference (zero_params,
    train.cpp:67-72)."""
    params = []
    for l, (d_in, d_out, _, shape) in enumerate(layer_dims(kind, layers, in_dim, hidden, classes)):
        if kind == SGC:
            params.append([np.zeros(shape), np.zeros(d_out)])
            continue
        a = np.sqrt(6.0 / (d_in + d_out))
        base = seed_for(seed, l)
        n = shape[0] * shape[1]
        u = np.array([mix64((base + i) & ((1 << 64) - 1)) >> 11 for i in range(n)], np.float64) * 2.0 ** -53
        params.append([((2.0 * u - 1.0) * a).reshape(shape), np.zeros(d_out)])
    return params


def flatten(params):
    return np.concatenate([np.concatenate([W.ravel(), b]) for W, b in params])


def unflatten(flat, like):
    out, k = [], 0
    for W, b in like:
        w = flat[k:k + W.size].reshape(W.shape); k += W.size
        bb = flat[k:k + b.size]; k += b.size
        out.append([w.copy(), bb.copy()])
    return out


def forward(kind, params, G: Graph, X, agg_first_flags):
    """Returns (H list incl. input at 0, Z list, aux list)."""
    H = [np.asarray(X, np.float64)]
    Zs, aux = [], []
    L = len(params)
    for l, (W, b) in enumerate(params):
        h = H[-1]
        if kind == GCN:
            dinv = 1.0 / np.sqrt(1.0 + G.deg)
            A_h = G.aggregate(h, "gcn", True, pre=dinv)
            Z = A_h @ W.T + b
            aux.append(A_h)
        elif kind == GIN:
            A_h = G.aggregate(h, "none", True)
            Z = A_h @ W.T + b
            aux.append(A_h)
        elif kind == SGC:
            A_h = G.aggregate(h, "sgc", True)  # sgc_propagate, one hop (train.cpp:49-65)
            Z = A_h @ W.T + b
            aux.append(A_h)
        else:
            m = G.aggregate(h, "mean", False)
            d_out = b.size
            if agg_first_flags[l]:
                d_in = h.shape[1]
                Ws, Wn = W[:, :d_in], W[:, d_in:]
            else:
                Ws, Wn = W[:d_out], W[d_out:]
            Z = h @ Ws.T + m @ Wn.T + b
            aux.append(m)
        Zs.append(Z)
        H.append(np.maximum(Z, 0.0) if l + 1 < L else Z)
    return H, Zs, aux


def loss_and_dlogits(Z, labels, train_rows):
    rows = np.asarray(train_rows, np.int64)
    dZ = np.zeros_like(Z)
    if rows.size == 0:
        return 0.0, dZ
    z = Z[rows]
    m = z.max(axis=1, keepdims=True)
    e = np.exp(z - m)
    s = e.sum(axis=1, keepdims=True)
    y = np.asarray(labels, np.int64)[rows]
    loss = float(np.mean(m[:, 0] + np.log(s[:, 0]) - z[np.arange(rows.size), y]))
    p = e / s
    p[np.arange(rows.size), y] -= 1.0
    dZ[rows] = p / rows.size
    return loss, dZ


def backward(kind, params, G: Graph, H, Zs, aux, dZ_last, agg_first_flags):
    grads = [None] * len(params)
    dZ = dZ_last
    for l in range(len(params) - 1, -1, -1):
        W, b = params[l]
        h = H[l]
        db = dZ.sum(axis=0)
        if kind in (GCN, GIN, SGC):
            dW = dZ.T @ aux[l]
            dA = dZ @ W
            if kind == GCN:
                dinv = 1.0 / np.sqrt(1.0 + G.deg)
                dh = G.aggregate(dA, "gcn", True, pre=dinv)
            elif kind == SGC:  # transpose of D~^-1 (A+I): (A+I) D~^-1
                dh = G.aggregate(dA, "none", True, pre=1.0 / (1.0 + G.deg))
            else:
                dh = G.aggregate(dA, "none", True)
        else:
            d_out = b.size
            d_in = h.shape[1]
            m = aux[l]
            if agg_first_flags[l]:
                Ws, Wn = W[:, :d_in], W[:, d_in:]
                dW = np.concatenate([dZ.T @ h, dZ.T @ m], axis=1)
            else:
                Ws, Wn = W[:d_out], W[d_out:]
                dW = np.concatenate([dZ.T @ h, dZ.T @ m], axis=0)
            dm = dZ @ Wn
            inv = np.where(G.deg > 0, 1.0 / np.maximum(G.deg, 1), 0.0)
            dh = dZ @ Ws + G.aggregate(dm, "none", False, pre=inv)
        grads[l] = [dW, db]
        if l > 0:
            dZ = dh * (Zs[l - 1] > 0)
    return grads


@dataclass
class OracleShard:
    G: Graph
    X: np.ndarray
    labels: np.ndarray
    train_rows: np.ndarray
    val_rows: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    test_rows: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))


class Replica:
    def __init__(self, kind, params, optimizer=ADAM, lr=0.01, beta1=0.9, beta2=0.999, eps=1e-8):
        self.kind = kind
        self.params = [[W.copy(), b.copy()] for W, b in params]
        self.opt = optimizer
        self.lr, self.b1, self.b2, self.eps = lr, beta1, beta2, eps
        flat = flatten(self.params)
        self.m = np.zeros_like(flat)
        self.v = np.zeros_like(flat)
        self.t = 0

    def flags(self, in_dim):
        dims = []
        d = in_dim
        for W, b in self.params:
            dims.append((d, b.size))
            d = b.size
        return [(di <= do) if self.kind == SAGE else (di < do) for di, do in dims]

    def forward_backward(self, sh: OracleShard):
        fl = self.flags(sh.X.shape[1])
        H, Zs, aux = forward(self.kind, self.params, sh.G, sh.X, fl)
        loss, dZ = loss_and_dlogits(Zs[-1], sh.labels, sh.train_rows)
        grads = backward(self.kind, self.params, sh.G, H, Zs, aux, dZ, fl)
        return loss, H, Zs, grads

    def step(self, sh: OracleShard):
        loss, H, Zs, grads = self.forward_backward(sh)
        g = flatten(grads)
        p = flatten(self.params)
        self.t += 1
        if self.opt == ADAM:
            self.m = self.b1 * self.m + (1 - self.b1) * g
            self.v = self.b2 * self.v + (1 - self.b2) * g * g
            mh = self.m / (1 - self.b1 ** self.t)
            vh = self.v / (1 - self.b2 ** self.t)
            p = p - self.lr * mh / (np.sqrt(vh) + self.eps)
        else:
            p = p - self.lr * g
        self.params = unflatten(p, self.params)
        return loss


def sync_weights(counts):
    """train.cpp:139-152."""
    counts = [int(c) for c in counts]
    total = sum(counts)
    if not counts or total == 0:
        raise ValueError("model averaging requires a nonzero training-node count")
    alpha = [c / total for c in counts[:-1]]
    alpha.append(1.0 - sum(alpha))
    return alpha


def model_average(params_list, counts):
    """train.cpp:154-172: sum_i alpha_i theta_i from zero, in partition order."""
    alpha = sync_weights(counts)
    flat = np.zeros_like(flatten(params_list[0]))
    for a, p in zip(alpha, params_list):
        flat = flat + a * flatten(p)
    return unflatten(flat, params_list[0])


def micro_f1(Z, labels, rows):
    rows = np.asarray(rows, np.int64)
    pred = np.argmax(Z[rows], axis=1)  # first maximum, like Eigen maxCoeff
    tp = int(np.sum(pred == np.asarray(labels)[rows]))
    miss = rows.size - tp
    den = 2 * tp + 2 * miss
    return 0.0 if den == 0 else 2.0 * tp / den


def distributed_train(kind, shards: List[OracleShard], sync_interval, epochs, layers, hidden, classes, seed,
                      optimizer=ADAM, lr=0.01, global_shard: OracleShard | None = None):
    """Per-partition full-batch training with averaging every s local iterations.
    Returns dict(params, losses per epoch, history [(epoch, syncs, val, test)])."""
    in_dim = shards[0].X.shape[1]
    shared = init_params(kind, layers, in_dim, hidden, classes, seed)
    reps = [Replica(kind, shared, optimizer, lr) for _ in shards]
    counts = [len(s.train_rows) for s in shards]
    alpha = sync_weights(counts)
    losses, hist = [], []
    done, ops = 0, 0
    while done < epochs:
        chunk = min(sync_interval, epochs - done)
        for r in reps:
            r.params = [[W.copy(), b.copy()] for W, b in shared]
        for _ in range(chunk):
            ep_loss = 0.0
            for a, r, s in zip(alpha, reps, shards):
                ep_loss += a * r.step(s)
            losses.append(ep_loss)
        shared = model_average([r.params for r in reps], counts)
        done += chunk
        ops += 1
        if global_shard is not None:
            fl = Replica(kind, shared).flags(in_dim)
            H, Zs, _ = forward(kind, shared, global_shard.G, global_shard.X, fl)
            vf = micro_f1(Zs[-1], global_shard.labels, global_shard.val_rows) if len(global_shard.val_rows) else 0.0
            tf = micro_f1(Zs[-1], global_shard.labels, global_shard.test_rows) if len(global_shard.test_rows) else 0.0
            hist.append((done, ops, vf, tf))
    return dict(params=shared, losses=losses, history=hist, averaging_ops=ops)


def shard_from_ref(rs) -> OracleShard:
    """OracleShard from oracle.ref.TrainingData.shard() (load_training_data,
    train.cpp:216-287, as the compiled reference built it)."""
    rows = rs.labels.size
    return OracleShard(Graph.from_csr(rs.offsets, rs.neighbors, rows), np.asarray(rs.features, np.float64),
                       rs.labels.astype(np.int64), rs.train_rows.astype(np.int64),
                       rs.val_rows.astype(np.int64), rs.test_rows.astype(np.int64))
