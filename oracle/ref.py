"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracle.

``oracle/_ref/libgnnpart_ref.so`` is the UNMODIFIED reference library
(/root/reference/proj/src/*.cpp) built by ``oracle/Makefile`` with the Eigen
shim.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
cpu_baseline / ``--impl reference`` legs may import this module; the product
package never does.

Every function mirrors the reference function named in its docstring and
raises ``RefError`` with the reference's exit-code convention (2 = ConfigError,
3 = DataError, 4 = other; proj/tools/gnnpart.cpp:387-399).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libgnnpart_ref.so")


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(
                f"oracle library missing: {LIB_PATH} (run `make -C oracle` where /root/reference exists)")
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_td_load.restype = C.c_void_p
        _lib.ref_td_free.argtypes = [C.c_void_p]
        _lib.ref_td_num_shards.argtypes = [C.c_void_p]
        _lib.ref_seed_for.restype = C.c_uint64
        _lib.ref_seed_for.argtypes = [C.c_uint64, C.c_uint64]
    return _lib


def _check(rc: int):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def seed_for(seed: int, stream: int) -> int:
    """common.hpp:37-39."""
    return int(lib().ref_seed_for(seed, stream))


def build_adjacency(rows: int, pairs: np.ndarray):
    """train.cpp:30-47 -> (offsets u32[rows+1], neighbors u32[nnz])."""
    pairs = np.ascontiguousarray(pairs, dtype=np.uint32).reshape(-1, 2)
    nnz = int(pairs.shape[0] * 2 - np.count_nonzero(pairs[:, 0] == pairs[:, 1]))
    offsets = np.zeros(rows + 1, np.uint32)
    nbrs = np.zeros(max(nnz, 1), np.uint32)
    _check(lib().ref_build_adjacency(C.c_uint32(rows), _p(pairs), C.c_uint64(pairs.shape[0]),
                                     _p(offsets), _p(nbrs), C.c_uint64(nbrs.size)))
    return offsets, nbrs[:nnz]


def sgc_propagate(offsets: np.ndarray, nbrs: np.ndarray, x: np.ndarray, hops: int) -> np.ndarray:
    """train.cpp:49-65 (f64)."""
    offsets = np.ascontiguousarray(offsets, np.uint32)
    nbrs = np.ascontiguousarray(nbrs, np.uint32)
    x = np.ascontiguousarray(x, np.float64)
    rows, dim = x.shape
    out = np.empty_like(x)
    _check(lib().ref_sgc_propagate(C.c_uint32(rows), _p(offsets), _p(nbrs), _p(x), C.c_uint32(dim),
                                   C.c_uint32(hops), _p(out)))
    return out


def sgc_propagate_colmajor(offsets, nbrs, x_colmajor: np.ndarray, rows: int, dim: int, hops: int):
    out = np.empty_like(x_colmajor)
    _check(lib().ref_sgc_propagate_colmajor(C.c_uint32(rows), _p(offsets), _p(nbrs), _p(x_colmajor),
                                            C.c_uint32(dim), C.c_uint32(hops), _p(out)))
    return out


def softmax_loss(W, b, x, y) -> float:
    """train.cpp:74-84."""
    W = np.ascontiguousarray(W, np.float64); b = np.ascontiguousarray(b, np.float64)
    x = np.ascontiguousarray(x, np.float64); y = np.ascontiguousarray(y, np.int32)
    out = C.c_double()
    _check(lib().ref_softmax_loss(_p(W), _p(b), C.c_uint32(W.shape[0]), C.c_uint32(W.shape[1]), _p(x),
                                  C.c_uint64(x.shape[0]), _p(y), C.byref(out)))
    return out.value


def softmax_gradient(W, b, x, y):
    """train.cpp:86-94 -> (gW [dim x C], gb [C])."""
    W = np.ascontiguousarray(W, np.float64); b = np.ascontiguousarray(b, np.float64)
    x = np.ascontiguousarray(x, np.float64); y = np.ascontiguousarray(y, np.int32)
    gW = np.empty_like(W); gb = np.empty_like(b)
    _check(lib().ref_softmax_gradient(_p(W), _p(b), C.c_uint32(W.shape[0]), C.c_uint32(W.shape[1]),
                                      _p(x), C.c_uint64(x.shape[0]), _p(y), _p(gW), _p(gb)))
    return gW, gb


def train_epochs(W, b, x, labels, train_rows, lr, batch, epoch_begin, epoch_end, seed):
    """train.cpp:96-128; returns updated (W, b) copies."""
    W = np.array(W, np.float64, order="C"); b = np.array(b, np.float64)
    x = np.ascontiguousarray(x, np.float64); labels = np.ascontiguousarray(labels, np.int32)
    tr = np.ascontiguousarray(train_rows, np.uint32)
    _check(lib().ref_train_epochs(_p(W), _p(b), C.c_uint32(W.shape[0]), C.c_uint32(W.shape[1]), _p(x),
                                  C.c_uint64(x.shape[0]), _p(labels), _p(tr), C.c_uint64(tr.size),
                                  C.c_double(lr), C.c_uint32(batch), C.c_uint64(epoch_begin),
                                  C.c_uint64(epoch_end), C.c_uint64(seed)))
    return W, b


def sync_weights(counts) -> np.ndarray:
    """train.cpp:139-152."""
    counts = np.ascontiguousarray(counts, np.uint64)
    alpha = np.zeros(counts.size, np.float64)
    _check(lib().ref_sync_weights(_p(counts), C.c_uint32(counts.size), _p(alpha)))
    return alpha


def model_average(Ws, bs, counts):
    """train.cpp:154-172."""
    Ws = np.ascontiguousarray(Ws, np.float64); bs = np.ascontiguousarray(bs, np.float64)
    counts = np.ascontiguousarray(counts, np.uint64)
    n, dim, Cn = Ws.shape
    W = np.empty((dim, Cn)); b = np.empty(Cn)
    _check(lib().ref_model_average(C.c_uint32(n), C.c_uint32(dim), C.c_uint32(Cn), _p(Ws), _p(bs),
                                   _p(counts), _p(W), _p(b)))
    return W, b


def evaluate_micro_f1(W, b, x, labels, mask) -> float:
    """train.cpp:174-198."""
    W = np.ascontiguousarray(W, np.float64); b = np.ascontiguousarray(b, np.float64)
    x = np.ascontiguousarray(x, np.float64); labels = np.ascontiguousarray(labels, np.int32)
    mask = np.ascontiguousarray(mask, np.uint32)
    out = C.c_double()
    _check(lib().ref_evaluate_micro_f1(_p(W), _p(b), C.c_uint32(W.shape[0]), C.c_uint32(W.shape[1]),
                                       _p(x), C.c_uint64(x.shape[0]), _p(labels), _p(mask),
                                       C.c_uint64(mask.size), C.byref(out)))
    return out.value


def partition(input_path, out_dir, partitions, *, nodes="", features="", algo="spring", fmt="",
              add_reverse=False, beta=1.05, tau_vol=0, lam=1.1, balance_slack=0.0, hops=1,
              no_completion=False, shuffle_isolated=False, seed=0):
    """The `gnnpart partition` handler (tools/gnnpart.cpp:61-109, :254-268)."""
    _check(lib().ref_partition(str(input_path).encode(), fmt.encode(), int(add_reverse),
                               str(nodes).encode(), str(features).encode(), algo.encode(),
                               C.c_uint32(partitions), C.c_double(beta), C.c_uint64(tau_vol),
                               C.c_double(lam), C.c_double(balance_slack), C.c_uint32(hops),
                               int(no_completion), int(shuffle_isolated), C.c_uint64(seed),
                               str(out_dir).encode()))


def spring_homes(input_path, num_ids, partitions, beta=1.05, tau_vol=0, seed=0, add_reverse=False):
    home = np.full(num_ids, 0xFFFFFFFF, np.uint32)
    _check(lib().ref_spring_homes(str(input_path).encode(), int(add_reverse), C.c_uint32(partitions),
                                  C.c_double(beta), C.c_uint64(tau_vol), C.c_uint64(seed), _p(home),
                                  C.c_uint64(num_ids)))
    return home


def compute_degrees(input_path, capacity, add_reverse=False):
    """GraphIndex of edge_stream.cpp:192-215: (dense_to_ext, degree, num_edges, num_self_loops)."""
    d2e = np.zeros(max(capacity, 1), np.uint64)
    deg = np.zeros(max(capacity, 1), np.uint32)
    n = C.c_uint64(); m = C.c_uint64(); sl = C.c_uint64()
    _check(lib().ref_compute_degrees(str(input_path).encode(), int(add_reverse), _p(d2e), _p(deg),
                                     C.c_uint64(capacity), C.byref(n), C.byref(m), C.byref(sl)))
    return d2e[:n.value], deg[:n.value], m.value, sl.value


def artifact_replication_factor(d):
    """metrics.cpp:9-12 over read_partitions (store.cpp:269-333); also the manifest's value."""
    rf = C.c_double(); mrf = C.c_double()
    _check(lib().ref_artifact_replication_factor(str(d).encode(), C.byref(rf), C.byref(mrf)))
    return rf.value, mrf.value


def write_synth(out_dir, nodes, edges, classes, dim, mixing=0.2, seed=1, binary=True):
    """synth.cpp DC-SBM dataset (alternate generator)."""
    _check(lib().ref_write_synth(C.c_uint64(nodes), C.c_uint64(edges), C.c_uint32(classes),
                                 C.c_uint32(dim), C.c_double(mixing), C.c_uint64(seed),
                                 str(out_dir).encode(), int(binary)))


@dataclass
class RefShard:
    offsets: np.ndarray
    neighbors: np.ndarray
    features: np.ndarray
    labels: np.ndarray
    train_rows: np.ndarray
    val_rows: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))
    test_rows: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


class TrainingData:
    """train.cpp:216-287 load_training_data, held by the oracle library."""

    def __init__(self, artifact_dir, input_override="", features_override=""):
        h = lib().ref_td_load(str(artifact_dir).encode(), str(input_override).encode(),
                              str(features_override).encode())
        if not h:
            raise RefError(3, lib().ref_last_error().decode())
        self._h = C.c_void_p(h)
        self.num_shards = lib().ref_td_num_shards(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            lib().ref_td_free(self._h)
            self._h = None

    def shard(self, s: int, with_features: bool = True) -> RefShard:
        """s = -1 is the global shard."""
        rows = C.c_uint64(); nnz = C.c_uint64(); dim = C.c_uint32()
        ntr = C.c_uint64(); nva = C.c_uint64(); nte = C.c_uint64()
        _check(lib().ref_td_shard_dims(self._h, s, C.byref(rows), C.byref(nnz), C.byref(dim),
                                       C.byref(ntr), C.byref(nva), C.byref(nte)))
        off = np.zeros(rows.value + 1, np.uint32)
        nb = np.zeros(max(nnz.value, 1), np.uint32)
        feats = np.zeros((rows.value, dim.value), np.float64) if with_features else None
        lab = np.zeros(max(rows.value, 1), np.int32)
        tr = np.zeros(max(ntr.value, 1), np.uint32)
        va = np.zeros(max(nva.value, 1), np.uint32)
        te = np.zeros(max(nte.value, 1), np.uint32)
        _check(lib().ref_td_shard_export(self._h, s, _p(off), _p(nb),
                                         _p(feats) if with_features else None, _p(lab), _p(tr),
                                         _p(va), _p(te)))
        return RefShard(off, nb[:nnz.value], feats, lab[:rows.value], tr[:ntr.value],
                        va[:nva.value], te[:nte.value])

    def distributed_train(self, workers, sync_interval, epochs=100, lr=0.01, batch=512,
                          prop_hops=2, seed=0, dim=None, classes=None):
        """train.cpp:289-340; returns dict(W, b, history, averaging_ops)."""
        if dim is None or classes is None:
            g = self.shard(-1, with_features=False)
            classes = int(g.labels.max()) + 1 if g.labels.size else 1
            d = C.c_uint64(); r = C.c_uint64(); dd = C.c_uint32(); a = C.c_uint64(); b_ = C.c_uint64(); c_ = C.c_uint64()
            _check(lib().ref_td_shard_dims(self._h, -1, C.byref(r), C.byref(d), C.byref(dd),
                                           C.byref(a), C.byref(b_), C.byref(c_)))
            dim = dd.value
        W = np.zeros((dim, classes)); b = np.zeros(classes)
        cap = (epochs + max(sync_interval, 1) - 1) // max(sync_interval, 1) + 1
        he = np.zeros(cap, np.uint64); hs = np.zeros(cap, np.uint64)
        hv = np.zeros(cap); ht = np.zeros(cap)
        dim_o = C.c_uint32(); cls_o = C.c_uint32(); nh = C.c_uint64(); ops = C.c_uint64()
        _check(lib().ref_td_distributed_train(self._h, C.c_uint32(workers), C.c_uint32(sync_interval),
                                              C.c_uint32(epochs), C.c_double(lr), C.c_uint32(batch),
                                              C.c_uint32(prop_hops), C.c_uint64(seed), _p(W), _p(b),
                                              C.byref(dim_o), C.byref(cls_o), _p(he), _p(hs), _p(hv),
                                              _p(ht), C.c_uint64(cap), C.byref(nh), C.byref(ops)))
        n = nh.value
        return dict(W=W, b=b, history=list(zip(he[:n].tolist(), hs[:n].tolist(), hv[:n].tolist(),
                                                ht[:n].tolist())), averaging_ops=ops.value)
