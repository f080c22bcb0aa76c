"""Synthetic inputs and the data formats either side of the training path.

* ``rmat_edges`` — RMAT(a,b,c,d) edge stream with E unique undirected pairs,
  no self-loops, first-seen orientation kept, ids compacted to 0..|V|-1 by
  rank among the seen raw ids.
* ``node_meta`` / ``class_features`` — the reference generator's label, role
  and feature scheme (proj/src/synth.cpp:135-148, :172-187): roles from split
  fractions over a shuffled order; features = class mean N(0,1)*signal +
  N(0, noise^2).  Labels are balanced id-rank buckets floor(cid*C/|V|).
* ``write_dataset`` — edges.bin (EDG1, edge_stream.cpp:174-183), nodes.tsv
  (write_node_meta, store.cpp:142-154) and features.bin (FEA1, store.cpp:15-23).
* ``complete_edges`` — 1-hop neighbour completion (completion.cpp:130-146 +
  PartitionBuilder :18-58) vectorised with NumPy: edge -> home(u) and, if
  different, home(v), stream order kept; node tables = owned nodes + edge
  endpoints, ascending external id, roles on owners only.  The per-partition
  unordered-pair dedup of the reference is a no-op on duplicate-free streams,
  which ``rmat_edges`` guarantees (checked).
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import List

import numpy as np

MASK64 = (1 << 64) - 1


def mix64(x: int) -> int:
    """common.hpp:27-32."""
    x = (x + 0x9E3779B97F4A7C15) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def seed_for(seed: int, stream: int) -> int:
    """common.hpp:37-39."""
    return mix64(seed ^ mix64((stream + 0x51ED2701) & MASK64))


def _mix64_np(x):
    """common.hpp:27-32 on uint64 arrays (wrapping arithmetic)."""
    x = x + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def _thr(p):
    return np.uint64(int(min(p * 4294967296.0, 4294967295.0)))


def _rmat_draw(base, idx, scale, a, b, c):
    """Quadrant choices of candidates idx (uint64 array): counter-based stream,
    word j of candidate i = splitmix64(base + 16 i + j//2), 32 bits per level."""
    ta, tab, tabc = _thr(a), _thr(a + b), _thr(a + b + c)
    s = np.zeros(idx.size, np.uint64)
    d = np.zeros(idx.size, np.uint64)
    word = None
    for level in range(scale):
        if level % 2 == 0:
            word = _mix64_np(np.uint64(base) + np.uint64(16) * idx + np.uint64(level >> 1))
        r = (word >> np.uint64(32)) if level & 1 else (word & np.uint64(0xFFFFFFFF))
        bs = r >= tab
        bd = ((r >= ta) & (r < tab)) | (r >= tabc)
        sh = np.uint64(scale - 1 - level)
        s |= bs.astype(np.uint64) << sh
        d |= bd.astype(np.uint64) << sh
    return s, d


def rmat_edges_numpy(scale: int, num_edges: int, a=0.57, b=0.19, c=0.19, seed=1):
    """Pure NumPy statement of the generator (checker for the C++ one)."""
    base = seed_for(seed, 0x3A7)
    n_cand = num_edges + num_edges * 3 // 10 + 1024
    while True:
        idx = np.arange(n_cand, dtype=np.uint64)
        s, d = _rmat_draw(base, idx, scale, a, b, c)
        valid = s != d
        key = (np.minimum(s, d) << np.uint64(32)) | np.maximum(s, d)
        vidx = idx[valid]
        _, first = np.unique(key[valid], return_index=True)
        if first.size >= num_edges:
            break
        n_cand = n_cand + n_cand // 2
    chosen = np.sort(vidx[first])[:num_edges]
    s, d = _rmat_draw(base, chosen, scale, a, b, c)
    seen = np.unique(np.concatenate([s, d]))
    e = np.empty((num_edges, 2), np.uint64)
    e[:, 0] = np.searchsorted(seen, s)
    e[:, 1] = np.searchsorted(seen, d)
    return e, int(seen.size), seen


def rmat_edges(scale: int, num_edges: int, a=0.57, b=0.19, c=0.19, seed=1):
    """RMAT stream via the parallel C++ generator (catgnn_synth_rmat), identical
    to rmat_edges_numpy.  Returns (edges uint64 [E,2] compacted, num_nodes, None)."""
    import ctypes as C
    from ._lib import check, lib
    e = np.empty((num_edges, 2), np.uint64)
    n = C.c_uint64()
    check(lib.catgnn_synth_rmat(C.c_uint32(scale), C.c_uint64(num_edges), C.c_double(a), C.c_double(b),
                                C.c_double(c), C.c_uint64(seed), e.ctypes.data_as(C.c_void_p), C.byref(n)))
    return e, int(n.value), None


def node_meta(num_nodes: int, classes: int, train_frac: float, val_frac: float, test_frac: float, seed: int):
    """labels int32 (id-rank buckets) and roles uint8 (0 none, 1 train, 2 val, 3 test)."""
    cid = np.arange(num_nodes, dtype=np.uint64)
    labels = ((cid * np.uint64(classes)) // np.uint64(max(num_nodes, 1))).astype(np.int32)
    rng = np.random.Generator(np.random.PCG64(seed_for(seed, 0x57A7)))
    order = rng.permutation(num_nodes)
    n_tr = int(train_frac * num_nodes); n_va = int(val_frac * num_nodes); n_te = int(test_frac * num_nodes)
    roles = np.zeros(num_nodes, np.uint8)
    roles[order[:n_tr]] = 1
    roles[order[n_tr:n_tr + n_va]] = 2
    roles[order[n_tr + n_va:n_tr + n_va + n_te]] = 3
    return labels, roles


def class_features(labels: np.ndarray, dim: int, classes: int, seed: int, signal=1.0, noise=2.0,
                   block=1 << 16) -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed_for(seed, 0xFEA7)))
    means = (rng.standard_normal((classes, dim)) * signal).astype(np.float32)
    n = labels.size
    out = np.empty((n, dim), np.float32)
    for i in range(0, n, block):
        j = min(n, i + block)
        out[i:j] = rng.standard_normal((j - i, dim), dtype=np.float32) * np.float32(noise)
        out[i:j] += means[labels[i:j]]
    return out


ROLE_NAMES = {0: "none", 1: "train", 2: "val", 3: "test"}


def write_dataset(d: str, edges: np.ndarray, labels: np.ndarray, roles: np.ndarray,
                  features: np.ndarray | None):
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "edges.bin"), "wb") as f:
        f.write(b"EDG1")
        np.ascontiguousarray(edges, np.uint64).tofile(f)
    names = np.array([ROLE_NAMES[i] for i in range(4)])
    lines = [f"{i}\t{int(l)}\t{names[r]}" for i, (l, r) in enumerate(zip(labels.tolist(), roles.tolist()))]
    with open(os.path.join(d, "nodes.tsv"), "w") as f:
        f.write("\n".join(lines) + ("\n" if lines else ""))
    if features is not None:
        with open(os.path.join(d, "features.bin"), "wb") as f:
            f.write(b"FEA1")
            f.write(np.uint64(features.shape[0]).tobytes())
            f.write(np.uint32(features.shape[1]).tobytes())
            f.write(np.uint32(1).tobytes())
            np.ascontiguousarray(features, np.float32).tofile(f)


@dataclass
class Part:
    edges: np.ndarray   # [E_s, 2] external ids, stream order
    ext: np.ndarray     # ascending external ids
    owner: np.ndarray   # uint8
    role: np.ndarray    # uint8 (owners only)

    @property
    def rows(self):
        return int(self.ext.size)


def complete_edges(edges: np.ndarray, home: np.ndarray, roles: np.ndarray, p: int) -> List[Part]:
    """1-hop completion (completion.cpp:130-146) for a duplicate-free stream."""
    n = home.size
    u = edges[:, 0].astype(np.int64); v = edges[:, 1].astype(np.int64)
    hu = home[u]; hv = home[v]
    parts = []
    for s in range(p):
        m = (hu == s) | (hv == s)
        es = edges[m]
        present = np.zeros(n, bool)
        present[es[:, 0].astype(np.int64)] = True
        present[es[:, 1].astype(np.int64)] = True
        present[home == s] = True
        ext = np.flatnonzero(present).astype(np.uint64)
        owner = (home[ext.astype(np.int64)] == s).astype(np.uint8)
        role = np.where(owner == 1, roles[ext.astype(np.int64)], 0).astype(np.uint8)
        parts.append(Part(np.ascontiguousarray(es), ext, owner, role))
    return parts


def replication_factor(parts: List[Part], num_nodes: int) -> float:
    """metrics.cpp:9-12."""
    return float(sum(p.rows for p in parts)) / float(num_nodes)
