"""Host-side mirror of the reference training API (namespace ``gnnpart``).

Same names, argument meaning and error behaviour as
/root/reference/proj/include/gnnpart/train.hpp, backed by the B200 kernels in
libcatgnn.so through the C ABI (include/catgnn.h).  Parameters are float32
NumPy arrays (the device computes in float32 / TF32); shards live on the GPU.

    reference (train.hpp)               this module
    ---------------------               -----------
    build_adjacency        :26-27       build_adjacency(rows, edges) -> LocalAdjacency
    sgc_propagate          :31-32       sgc_propagate(shard, hops)   (shard holds adj + x)
    zero_params            :40          zero_params(dim, classes)
    softmax_loss           :50-51       softmax_loss(params, shard, rows)
    softmax_gradient       :53-55       softmax_gradient(params, shard, rows)
    train_epochs           :61-64       train_epochs(params, shard, cfg, begin, end, seed)
    train_local            :66-67       train_local(shard, cfg)
    sync_weights           :71          sync_weights(counts)
    model_average          :73-74       model_average(params_list, counts)
    evaluate_micro_f1      :78-81       evaluate_micro_f1(params, shard, mask_rows)
    load_training_data     :100-103     load_training_data(artifact_dir, input=, features=)
    distributed_train      :123-124     distributed_train(data, workers, sync_interval, cfg)
    replication_factor     metrics.hpp:46  replication_factor(artifact)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from ._lib import (ArtifactInfo, ConfigError, DataError, DistResult, InternalError, ShardInfo,
                   TrainConfig, check, lib)

__all__ = [
    "Context", "Artifact", "Shard", "LocalAdjacency", "ModelParams", "TrainConfig", "TrainingData",
    "SyncPoint", "DistTrainResult", "ConfigError", "DataError", "InternalError", "build_adjacency",
    "sgc_propagate", "zero_params", "softmax_loss", "softmax_gradient", "train_epochs", "train_local",
    "sync_weights", "model_average", "evaluate_micro_f1", "load_training_data", "distributed_train",
    "replication_factor", "default_context", "FeatureStore", "GraphPartition", "complete_edges", "GraphIndex", "compute_degrees",
]


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Context:
    """A device + CUDA stream (catgnn_ctx)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        h = C.c_void_p()
        check(lib.catgnn_ctx_create(device, C.c_void_p(stream) if stream else None, C.byref(h)))
        self.handle = h
        self.device = device

    def synchronize(self):
        check(lib.catgnn_ctx_synchronize(self.handle))

    @property
    def launches(self) -> int:
        return int(lib.catgnn_ctx_launch_count(self.handle))

    def wait_for(self, other: "Context"):
        """Order this context's later work after `other`'s work enqueued so far."""
        check(lib.catgnn_ctx_wait(self.handle, other.handle))

    def set_sm_budget(self, agg_sms: int = 0, gemm_sms: int = 0):
        """Persistent-grid SM budgets of this context's K2 / K3 launches (0 = all SMs)."""
        check(lib.catgnn_ctx_set_sm_budget(self.handle, int(agg_sms), int(gemm_sms)))

    def set_kernel_timing(self, enable: bool):
        check(lib.catgnn_ctx_set_kernel_timing(self.handle, int(enable)))

    def kernel_time(self):
        a = C.c_double(); an = C.c_uint64(); g = C.c_double(); gn = C.c_uint64()
        check(lib.catgnn_ctx_kernel_time(self.handle, C.byref(a), C.byref(an), C.byref(g), C.byref(gn)))
        return dict(agg_ms=a.value, agg_launches=an.value, gemm_ms=g.value, gemm_launches=gn.value)

    def kernel_records(self):
        """Per-label totals of the timed launches: {label: (ms_total, launches)}."""
        n = C.c_uint32()
        check(lib.catgnn_ctx_timing_record(self.handle, 0, None, 0, C.byref(n)))
        out = {}
        buf = C.create_string_buffer(512)
        for i in range(n.value):
            check(lib.catgnn_ctx_timing_record(self.handle, i, buf, 512, C.byref(n)))
            label, ms, cnt = buf.value.decode().split("\t")
            out[label] = (float(ms), int(cnt))
        return out

    def close(self):
        if getattr(self, "handle", None):
            lib.catgnn_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = Context(0)
    return _default_ctx


class Artifact:
    """Host view of a stored partition artifact (read_partitions, store.cpp:269-333)."""

    def __init__(self, directory: str):
        h = C.c_void_p()
        check(lib.catgnn_artifact_open(str(directory).encode(), C.byref(h)))
        self.handle = h
        self.directory = str(directory)
        info = ArtifactInfo()
        check(lib.catgnn_artifact_get_info(h, C.byref(info)))
        self.info = info
        self.num_partitions = info.num_partitions

    def part_counts(self, part: int):
        n = C.c_uint64(); o = C.c_uint64(); e = C.c_uint64()
        check(lib.catgnn_artifact_part_counts(self.handle, part, C.byref(n), C.byref(o), C.byref(e)))
        return n.value, o.value, e.value

    def replica_map(self, part: int):
        """(ext_ids u64, owner u8, role u8, home u32) in local row order."""
        n, _, _ = self.part_counts(part)
        ext = np.zeros(n, np.uint64); own = np.zeros(n, np.uint8)
        role = np.zeros(n, np.uint8); home = np.zeros(n, np.uint32)
        check(lib.catgnn_artifact_replica_map(self.handle, part, _ptr(ext), _ptr(own), _ptr(role), _ptr(home)))
        return ext, own, role, home

    def close(self):
        if getattr(self, "handle", None):
            lib.catgnn_artifact_close(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def replication_factor(artifact: Artifact) -> float:
    """metrics.cpp:9-12: sum of node records / |V| (f64)."""
    return artifact.info.replication_factor


@dataclass
class LocalAdjacency:
    """train.hpp:18-24 (offsets widened to u64)."""
    offsets: np.ndarray
    neighbors: np.ndarray

    def rows(self) -> int:
        return 0 if self.offsets.size == 0 else self.offsets.size - 1


class Shard:
    """Device-resident gnnpart::Shard (train.hpp:84-91)."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self.handle = handle
        self.ctx = ctx
        self._info = None

    # -- constructors ---------------------------------------------------
    @classmethod
    def from_edges(cls, rows: int, edges, features: Optional[np.ndarray] = None,
                   ctx: Optional[Context] = None) -> "Shard":
        ctx = ctx or default_context()
        pairs = np.ascontiguousarray(np.asarray(edges, dtype=np.uint32).reshape(-1, 2))
        feats = None
        dim = 0
        if features is not None:
            feats = np.ascontiguousarray(features, dtype=np.float32)
            dim = feats.shape[1]
        h = C.c_void_p()
        check(lib.catgnn_shard_create(ctx.handle, rows, _ptr(pairs), pairs.shape[0], _ptr(feats), dim,
                                      C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_artifact(cls, artifact: Artifact, part: int, input: str = "", features: str = "",
                      ctx: Optional[Context] = None) -> "Shard":
        ctx = ctx or default_context()
        h = C.c_void_p()
        check(lib.catgnn_shard_load(ctx.handle, artifact.handle, part, (input or "").encode(),
                                    (features or "").encode(), C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_part(cls, ext_ids, owner, role, labels, edges_ext, features, ctx=None) -> "Shard":
        ctx = ctx or default_context()
        ext = np.ascontiguousarray(ext_ids, np.uint64)
        own = np.ascontiguousarray(owner, np.uint8)
        rl = np.ascontiguousarray(role, np.uint8)
        lab = np.ascontiguousarray(labels, np.int32)
        ed = np.ascontiguousarray(np.asarray(edges_ext, np.uint64).reshape(-1, 2))
        feats = np.ascontiguousarray(features, np.float32) if features is not None else None
        dim = 0 if feats is None else feats.shape[1]
        h = C.c_void_p()
        check(lib.catgnn_shard_create_from_part(ctx.handle, ext.size, _ptr(ext), _ptr(own), _ptr(rl), _ptr(lab),
                                                _ptr(ed), ed.shape[0], _ptr(feats), dim, C.byref(h)))
        return cls(h, ctx)

    # -- accessors -------------------------------------------------------
    def halo_map(self, artifact: "Artifact"):
        """(home u32 per local row, halo row count), built on the shard's device."""
        home = np.zeros(self.rows, np.uint32)
        n = C.c_uint64()
        check(lib.catgnn_shard_halo_map(self.handle, artifact.handle, _ptr(home), C.byref(n)))
        return home, n.value

    def train_views(self):
        """(rows, nnz) of the train-row view and nnz of the train-neighbour view."""
        a = C.c_uint64(); b = C.c_uint64(); c = C.c_uint64()
        check(lib.catgnn_shard_train_views(self.handle, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    @property
    def info(self) -> ShardInfo:
        inf = ShardInfo()
        check(lib.catgnn_shard_get_info(self.handle, C.byref(inf)))
        return inf

    @property
    def rows(self) -> int:
        return int(self.info.rows)

    @property
    def dim(self) -> int:
        return int(self.info.dim)

    def adjacency(self) -> LocalAdjacency:
        inf = self.info
        off = np.zeros(inf.rows + 1, np.uint64)
        nb = np.zeros(max(inf.nnz, 1), np.uint32)
        check(lib.catgnn_csr_export(self.handle, _ptr(off), _ptr(nb)))
        return LocalAdjacency(off, nb[: inf.nnz])

    def set_labels(self, labels, train_rows=(), val_rows=(), test_rows=()):
        lab = np.ascontiguousarray(labels, np.int32)
        tr = np.ascontiguousarray(train_rows, np.uint32)
        va = np.ascontiguousarray(val_rows, np.uint32)
        te = np.ascontiguousarray(test_rows, np.uint32)
        check(lib.catgnn_shard_set_labels(self.handle, _ptr(lab), _ptr(tr), tr.size, _ptr(va), va.size,
                                          _ptr(te), te.size))

    def upload_features(self, features: np.ndarray):
        f = np.ascontiguousarray(features, np.float32)
        check(lib.catgnn_shard_upload_features(self.handle, _ptr(f), f.shape[1]))

    def set_feature_layout(self, split_only: bool):
        """catgnn_shard_set_feature_layout: gathers write only the bf16x3 copy."""
        check(lib.catgnn_shard_set_feature_layout(self.handle, int(split_only)))

    def gather_features(self, store: "FeatureStore"):
        """x[r] = F[ext_id(r)] on the device (train.cpp:277-283)."""
        check(lib.catgnn_shard_gather_features(self.handle, store.handle))

    def role_rows(self, role: int) -> np.ndarray:
        inf = self.info
        n = {1: inf.n_train, 2: inf.n_val, 3: inf.n_test}[role]
        out = np.zeros(max(n, 1), np.uint32)
        check(lib.catgnn_shard_role_rows(self.handle, role, _ptr(out)))
        return out[:n]

    @property
    def train_rows(self):
        return self.role_rows(1)

    @property
    def val_rows(self):
        return self.role_rows(2)

    @property
    def test_rows(self):
        return self.role_rows(3)

    @property
    def labels(self) -> np.ndarray:
        out = np.zeros(max(self.rows, 1), np.int32)
        check(lib.catgnn_shard_labels(self.handle, _ptr(out)))
        return out[: self.rows]

    def features(self, propagated: bool = False) -> np.ndarray:
        out = np.zeros((self.rows, self.dim), np.float32)
        check(lib.catgnn_shard_export_features(self.handle, 1 if propagated else 0, _ptr(out)))
        return out

    def close(self):
        if getattr(self, "handle", None):
            lib.catgnn_shard_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class GraphPartition:
    """GraphPartition (completion.hpp:31-34): edges (E x 2 ext ids, stream
    order), node table (ascending ext ids, owner flags, roles)."""
    edges: np.ndarray
    ext: np.ndarray
    owner: np.ndarray
    role: np.ndarray

    @property
    def rows(self) -> int:
        return int(self.ext.size)


class GraphIndex:
    """GraphIndex (edge_stream.hpp:104-128) built on the device by
    compute_degrees (edge_stream.cpp:192-215)."""

    def __init__(self, handle: C.c_void_p, ctx: Context):
        self.handle, self.ctx = handle, ctx
        n, m, sl = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(lib.catgnn_index_info(handle, C.byref(n), C.byref(m), C.byref(sl)))
        self.num_nodes, self.num_edges, self.num_self_loops = n.value, m.value, sl.value
        self.dense_to_ext = np.zeros(self.num_nodes, np.uint64)
        self.degree = np.zeros(self.num_nodes, np.uint32)
        check(lib.catgnn_index_export(handle, _ptr(self.dense_to_ext), _ptr(self.degree)))

    def close(self):
        if getattr(self, "handle", None):
            lib.catgnn_index_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def compute_degrees(edges, ctx: Optional[Context] = None) -> GraphIndex:
    """compute_degrees (edge_stream.cpp:192-215) over an in-memory stream."""
    ctx = ctx or default_context()
    e = np.ascontiguousarray(np.asarray(edges, np.uint64).reshape(-1, 2))
    h = C.c_void_p()
    check(lib.catgnn_index_build(ctx.handle, _ptr(e), e.shape[0], C.byref(h)))
    return GraphIndex(h, ctx)


def complete_edges_file(path: str, home, roles=None, partitions: Optional[int] = None, hops: int = 1,
                        add_reverse: bool = False, ctx: Optional[Context] = None) -> List[GraphPartition]:
    """complete_edges over an edge file (EDG1 streamed in chunks; dense ids)."""
    ctx = ctx or default_context()
    h = np.ascontiguousarray(home, np.uint32)
    r = None if roles is None else np.ascontiguousarray(roles, np.uint8)
    p = int(partitions if partitions is not None else (int(h.max()) + 1 if h.size else 0))
    c = C.c_void_p()
    check(lib.catgnn_complete_edges_file(ctx.handle, str(path).encode(), int(add_reverse), _ptr(h), _ptr(r),
                                         h.size, p, hops, C.byref(c)))
    return _completion_parts(c, p)


def _completion_parts(c, p) -> List[GraphPartition]:
    try:
        out = []
        for s in range(p):
            ne, nn = C.c_uint64(), C.c_uint64()
            check(lib.catgnn_completion_part_counts(c, s, C.byref(ne), C.byref(nn), None))
            pe = np.zeros((ne.value, 2), np.uint64)
            ext = np.zeros(nn.value, np.uint64)
            own = np.zeros(nn.value, np.uint8)
            rl = np.zeros(nn.value, np.uint8)
            check(lib.catgnn_completion_part(c, s, _ptr(pe), _ptr(ext), _ptr(own), _ptr(rl)))
            out.append(GraphPartition(pe, ext, own, rl))
        return out
    finally:
        lib.catgnn_completion_destroy(c)


def complete_edges(edges, home, roles=None, partitions: Optional[int] = None, hops: int = 1,
                   ctx: Optional[Context] = None, index: Optional[GraphIndex] = None) -> List[GraphPartition]:
    """complete_edges (completion.cpp:130-171) on the device.  Without `index`
    the external ids must be dense (home/roles indexed by ext id); with a
    GraphIndex any 64-bit ids work and home/roles are indexed by dense id."""
    ctx = ctx or default_context()
    e = np.ascontiguousarray(np.asarray(edges, np.uint64).reshape(-1, 2))
    h = np.ascontiguousarray(home, np.uint32)
    r = None if roles is None else np.ascontiguousarray(roles, np.uint8)
    p = int(partitions if partitions is not None else (int(h.max()) + 1 if h.size else 0))
    c = C.c_void_p()
    if index is None:
        check(lib.catgnn_complete_edges(ctx.handle, _ptr(e), e.shape[0], _ptr(h), _ptr(r), h.size, p, hops,
                                        C.byref(c)))
    else:
        if h.size != index.num_nodes:
            raise DataError("home map does not cover the node set")
        check(lib.catgnn_complete_edges_indexed(ctx.handle, index.handle, _ptr(e), e.shape[0], _ptr(h), _ptr(r),
                                                p, hops, C.byref(c)))
    try:
        out = []
        for s in range(p):
            ne, nn = C.c_uint64(), C.c_uint64()
            check(lib.catgnn_completion_part_counts(c, s, C.byref(ne), C.byref(nn), None))
            pe = np.zeros((ne.value, 2), np.uint64)
            ext = np.zeros(nn.value, np.uint64)
            own = np.zeros(nn.value, np.uint8)
            rl = np.zeros(nn.value, np.uint8)
            check(lib.catgnn_completion_part(c, s, _ptr(pe), _ptr(ext), _ptr(own), _ptr(rl)))
            out.append(GraphPartition(pe, ext, own, rl))
        return out
    finally:
        lib.catgnn_completion_destroy(c)


def probe_read_bandwidth(nbytes: int, passes: int = 20, ctx: Optional[Context] = None) -> float:
    """Device read bandwidth in GB/s (L2 when nbytes fits the 126 MB L2)."""
    ctx = ctx or default_context()
    out = C.c_double()
    check(lib.catgnn_probe_read_bandwidth(ctx.handle, int(nbytes), int(passes), C.byref(out)))
    return out.value


class FeatureStore:
    """Device copy of the global feature matrix (rows x dim f32, FEA1 row
    order) that shards gather their rows from by external id."""

    def __init__(self, rows: int, dim: int, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.rows, self.dim = int(rows), int(dim)
        h = C.c_void_p()
        check(lib.catgnn_features_create(self.ctx.handle, self.rows, self.dim, C.byref(h)))
        self.handle = h

    def upload(self, features: np.ndarray, row_begin: int = 0):
        f = features if (features.dtype == np.float32 and features.flags.c_contiguous) \
            else np.ascontiguousarray(features, np.float32)
        if f.ndim != 2 or f.shape[1] != self.dim:
            raise ConfigError(f"feature rows must be {self.dim} wide")
        check(lib.catgnn_features_upload(self.handle, _ptr(f), row_begin, f.shape[0]))

    def reset_deps(self):
        """Forget recorded upload / gather events (stream order from here on)."""
        check(lib.catgnn_features_reset_deps(self.handle))

    def allgather(self, comm, rows_per_rank: int):
        """In-place NCCL all-gather of every rank's row slice (see catgnn.h)."""
        check(lib.catgnn_features_allgather(self.handle, comm.handle, int(rows_per_rank)))

    def close(self):
        if getattr(self, "handle", None):
            lib.catgnn_features_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build_adjacency(rows: int, edges, ctx: Optional[Context] = None) -> LocalAdjacency:
    """train.cpp:30-47 on the device; bit-exact offsets/neighbors."""
    s = Shard.from_edges(rows, edges, None, ctx)
    try:
        return s.adjacency()
    finally:
        s.close()


def sgc_propagate(shard: Shard, hops: int) -> np.ndarray:
    """train.cpp:49-65: hops rounds of (x_i + sum_j x_j) / (1 + deg_i)."""
    check(lib.catgnn_sgc_propagate(shard.handle, hops))
    return shard.features(propagated=True)


@dataclass
class ModelParams:
    """train.hpp:34-38 (float32)."""
    weight: np.ndarray  # dim x classes
    bias: np.ndarray    # classes
    epochs_trained: int = 0

    def copy(self) -> "ModelParams":
        return ModelParams(self.weight.copy(), self.bias.copy(), self.epochs_trained)


def zero_params(dim: int, classes: int) -> ModelParams:
    """train.cpp:67-72."""
    return ModelParams(np.zeros((dim, classes), np.float32), np.zeros(classes, np.float32))


def _wb(p: ModelParams):
    p.weight = np.ascontiguousarray(p.weight, np.float32)
    p.bias = np.ascontiguousarray(p.bias, np.float32)
    return p.weight, p.bias


def softmax_loss(params: ModelParams, shard: Shard, rows) -> float:
    """train.cpp:74-84 over the given rows of the propagated features."""
    W, b = _wb(params)
    r = np.ascontiguousarray(rows, np.uint32)
    out = C.c_double()
    check(lib.catgnn_softmax_loss(shard.handle, _ptr(W), _ptr(b), W.shape[1], _ptr(r), r.size, C.byref(out)))
    return out.value


def softmax_gradient(params: ModelParams, shard: Shard, rows):
    """train.cpp:86-94 -> (grad_weight, grad_bias)."""
    W, b = _wb(params)
    r = np.ascontiguousarray(rows, np.uint32)
    gW = np.zeros_like(W); gb = np.zeros_like(b)
    check(lib.catgnn_softmax_gradient(shard.handle, _ptr(W), _ptr(b), W.shape[1], _ptr(r), r.size, _ptr(gW),
                                      _ptr(gb)))
    return gW, gb


def train_epochs(params, shards, cfg: TrainConfig, epoch_begin: int, epoch_end: int, seeds):
    """train.cpp:96-128.  params/shards/seeds may be lists: replicas train in one launch."""
    single = isinstance(params, ModelParams)
    plist = [params] if single else list(params)
    slist = [shards] if single else list(shards)
    seeds = [seeds] if single else list(seeds)
    if not plist:
        return params
    ws = [_wb(p)[0] for p in plist]
    bs = [p.bias for p in plist]
    n = len(plist)
    Wp = (C.c_void_p * n)(*[w.ctypes.data for w in ws])
    bp = (C.c_void_p * n)(*[b.ctypes.data for b in bs])
    sh = (C.c_void_p * n)(*[s.handle.value for s in slist])
    sd = np.ascontiguousarray(seeds, np.uint64)
    check(lib.catgnn_train_epochs(n, sh, Wp, bp, ws[0].shape[1], cfg.lr, cfg.batch, epoch_begin, epoch_end,
                                  _ptr(sd)))
    for p in plist:
        p.epochs_trained = epoch_end
    return params


def train_local(shard: Shard, cfg: TrainConfig) -> ModelParams:
    """train.cpp:130-137 via catgnn_train_local: zero_params(dim, max label + 1),
    then train_epochs over the shard's train rows with cfg.seed, on its
    features propagated cfg.prop_hops times (train-sim --compare-centralized,
    gnnpart.cpp:330-335, on the global shard)."""
    classes = C.c_uint32()
    check(lib.catgnn_train_local(shard.handle, C.byref(cfg), None, None, C.byref(classes)))
    p = zero_params(shard.dim, classes.value)
    check(lib.catgnn_train_local(shard.handle, C.byref(cfg), _ptr(p.weight), _ptr(p.bias), C.byref(classes)))
    p.epochs_trained = cfg.epochs
    return p


def sync_weights(counts) -> np.ndarray:
    """train.cpp:139-152."""
    c = np.ascontiguousarray(counts, np.uint64)
    a = np.zeros(c.size, np.float64)
    check(lib.catgnn_sync_weights(_ptr(c), c.size, _ptr(a)))
    return a


def model_average(params: List[ModelParams], counts, ctx: Optional[Context] = None) -> ModelParams:
    """train.cpp:154-172 (computed on the device)."""
    ctx = ctx or default_context()
    if not params or len(params) != len(counts):
        raise DataError("model averaging needs one training count per replica")
    shapes = {(p.weight.shape, p.bias.shape) for p in params}
    if len(shapes) != 1:
        raise DataError("model shapes differ across replicas")
    flat = [np.concatenate([np.asarray(p.weight, np.float32).ravel(), np.asarray(p.bias, np.float32)])
            for p in params]
    n = len(flat)
    ptrs = (C.c_void_p * n)(*[f.ctypes.data for f in flat])
    c = np.ascontiguousarray(counts, np.uint64)
    out = np.zeros_like(flat[0])
    check(lib.catgnn_model_average_host(ctx.handle, n, ptrs, out.size, _ptr(c), _ptr(out)))
    W = params[0].weight
    return ModelParams(out[: W.size].reshape(W.shape).copy(), out[W.size:].copy(), params[0].epochs_trained)


def evaluate_micro_f1(params: ModelParams, shard: Shard, mask_rows) -> float:
    """train.cpp:174-198 on the propagated features."""
    W, b = _wb(params)
    m = np.ascontiguousarray(mask_rows, np.uint32)
    out = C.c_double()
    check(lib.catgnn_evaluate_micro_f1(shard.handle, _ptr(W), _ptr(b), W.shape[1], _ptr(m), m.size, C.byref(out)))
    return out.value


@dataclass
class TrainingData:
    """train.hpp:93-96."""
    shards: List[Shard]
    global_: Shard
    artifact: Optional[Artifact] = None


def split_features(features: str, artifact_dir: str, out_dir: str, ctx: Optional[Context] = None) -> int:
    """store.cpp:97-116: part-<s>/features.bin for every partition of the
    artifact from the global FEA1 matrix (device row gather); returns the
    number of files written."""
    ctx = ctx or default_context()
    art = Artifact(artifact_dir)
    n = C.c_uint32()
    check(lib.catgnn_split_features(ctx.handle, art.handle, str(features).encode(), str(out_dir).encode(),
                                    C.byref(n)))
    return int(n.value)


def load_training_data(artifact_dir: str, input: str = "", features: str = "",
                       ctx: Optional[Context] = None, with_global: bool = True) -> TrainingData:
    """train.cpp:216-287: one device shard per partition plus the global shard."""
    ctx = ctx or default_context()
    art = Artifact(artifact_dir)
    g = Shard.from_artifact(art, -1, input, features, ctx) if with_global else None
    shards = [Shard.from_artifact(art, s, input, features, ctx) for s in range(art.num_partitions)]
    return TrainingData(shards, g, art)


@dataclass
class SyncPoint:
    epoch: int
    syncs: int
    val_f1: float
    test_f1: float


@dataclass
class DistTrainResult:
    params: ModelParams
    history: List[SyncPoint] = field(default_factory=list)
    averaging_ops: int = 0


def distributed_train(data: TrainingData, workers: int, sync_interval: int, cfg: TrainConfig) -> DistTrainResult:
    """train.cpp:289-340 on one device (workers are logical; p % q == 0)."""
    g = data.global_
    gi = g.info
    p = len(data.shards)
    W = np.zeros((gi.dim, gi.classes), np.float32)
    b = np.zeros(gi.classes, np.float32)
    cap = (cfg.epochs + max(sync_interval, 1) - 1) // max(sync_interval, 1) + 1
    he = np.zeros(cap, np.uint64); hs = np.zeros(cap, np.uint64)
    hv = np.zeros(cap, np.float64); ht = np.zeros(cap, np.float64)
    res = DistResult(W.ctypes.data, b.ctypes.data, 0, 0, he.ctypes.data, hs.ctypes.data, hv.ctypes.data,
                     ht.ctypes.data, cap, 0, 0)
    sh = (C.c_void_p * max(p, 1))(*[s.handle.value for s in data.shards])
    check(lib.catgnn_distributed_train(p, sh, g.handle, workers, sync_interval, C.byref(cfg), C.byref(res)))
    n = min(res.n_hist, cap)
    hist = [SyncPoint(int(he[i]), int(hs[i]), float(hv[i]), float(ht[i])) for i in range(n)]
    return DistTrainResult(ModelParams(W, b, cfg.epochs), hist, int(res.averaging_ops))
