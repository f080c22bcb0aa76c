"""GNN replicas (north-star layers) over the C ABI, and the partition-parallel
training loop with model averaging — the GNN counterpart of
gnnpart.distributed_train (proj/src/train.cpp:289-340).

One local iteration = one full-batch forward/backward/optimizer step on a
partition shard.  Every `sync_interval` iterations
the replicas are averaged with alpha_i = n_train_i / sum n_train
(train.cpp:139-172): in-process on one GPU (catgnn_model_average), or across
ranks with the alpha-prescaled NCCL all-reduce (catgnn_model_scale +
catgnn_model_allreduce).  Partitions are assigned to ranks cyclically
(PAPER.md:231), p % world == 0 (train.cpp:293-294).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from ._lib import GnnResult, GnnTrainConfig, ModelConfig, check, lib
from .gnnpart import Context, Shard, default_context

GCN, SAGE, GIN, SGC = 1, 2, 3, 4
KINDS = {"gcn": GCN, "sage": SAGE, "gin": GIN, "sgc": SGC}
SGD, ADAM = 0, 1


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class GNNModel:
    def __init__(self, kind, layers, in_dim, hidden, classes, optimizer=ADAM, lr=0.01, seed=0,
                 beta1=0.9, beta2=0.999, eps=1e-8, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        k = KINDS[kind] if isinstance(kind, str) else kind
        self.cfg = ModelConfig(k, layers, in_dim, hidden, classes, optimizer, lr, beta1, beta2, eps, seed)
        h = C.c_void_p()
        check(lib.catgnn_model_create(self.ctx.handle, C.byref(self.cfg), C.byref(h)))
        self.handle = h
        self.num_params = int(lib.catgnn_model_num_params(h))

    @classmethod
    def adopt(cls, handle: C.c_void_p, ctx: Context, cfg: ModelConfig) -> "GNNModel":
        """Wrap a model the library created (e.g. catgnn_gnn_distributed_train's result)."""
        m = cls.__new__(cls)
        m.ctx = ctx
        m.handle = handle
        m.num_params = int(lib.catgnn_model_num_params(handle))
        m.cfg = cfg
        return m

    def set_act_f16(self, on: bool):
        """fp16 aggregation inputs where safe (GCN backward, last-layer forward)."""
        check(lib.catgnn_model_set_act_f16(self.handle, int(bool(on))))

    def layer_shapes(self):
        out = []
        for l in range(self.cfg.layers):
            r = C.c_uint32(); c = C.c_uint32(); ow = C.c_uint64(); ob = C.c_uint64()
            check(lib.catgnn_model_layer_shape(self.handle, l, C.byref(r), C.byref(c), C.byref(ow), C.byref(ob)))
            out.append(((r.value, c.value), ow.value, ob.value))
        return out

    def get_params(self) -> np.ndarray:
        out = np.zeros(self.num_params, np.float32)
        check(lib.catgnn_model_get_params(self.handle, _ptr(out)))
        return out

    def set_params(self, flat):
        f = np.ascontiguousarray(flat, np.float32)
        assert f.size == self.num_params
        check(lib.catgnn_model_set_params(self.handle, _ptr(f)))

    def get_grads(self) -> np.ndarray:
        out = np.zeros(self.num_params, np.float32)
        check(lib.catgnn_model_get_grads(self.handle, _ptr(out)))
        return out

    def unflatten(self, flat):
        """Logical flat vector -> [[W, b], ...] per layer."""
        shapes = self.layer_shapes()
        res = []
        for i, (shape, ow, ob) in enumerate(shapes):
            end = shapes[i + 1][1] if i + 1 < len(shapes) else self.num_params
            res.append([flat[ow:ow + shape[0] * shape[1]].reshape(shape), flat[ob:end]])
        return res

    def copy_params_from(self, other: "GNNModel"):
        check(lib.catgnn_model_copy_params(self.handle, other.handle))

    def train_step(self, shard: Shard, want_loss: bool = True) -> Optional[float]:
        loss = C.c_double()
        check(lib.catgnn_model_train_step(self.handle, shard.handle, C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def last_loss(self) -> float:
        """Loss of the last train_step, read back now (one sync)."""
        loss = C.c_double()
        check(lib.catgnn_model_last_loss(self.handle, C.byref(loss)))
        return loss.value

    def last_loss_async(self, host_sum) -> int:
        """Enqueue the D2H copy of the last step's loss sum into host_sum (a
        pinned float64 buffer's address); returns the train-row count."""
        rows = C.c_uint64()
        check(lib.catgnn_model_last_loss_async(self.handle, C.cast(host_sum, C.POINTER(C.c_double)),
                                               C.byref(rows)))
        return int(rows.value)

    def forward_backward(self, shard: Shard) -> float:
        loss = C.c_double()
        check(lib.catgnn_model_forward_backward(self.handle, shard.handle, C.byref(loss)))
        return loss.value

    def forward(self, shard: Shard, logits: bool = False, role: int = 0):
        out = np.zeros((shard.rows, self.cfg.classes), np.float32) if logits else None
        f1 = C.c_double()
        check(lib.catgnn_model_forward(self.handle, shard.handle, _ptr(out) if logits else None, role,
                                       C.byref(f1) if role else None))
        return out, (f1.value if role else None)

    def export(self, layer: int, what: int, rows: int) -> np.ndarray:
        w = C.c_uint32()
        check(lib.catgnn_model_export(self.handle, layer, what, None, C.byref(w)))
        out = np.zeros((rows, w.value), np.float32)
        check(lib.catgnn_model_export(self.handle, layer, what, _ptr(out), C.byref(w)))
        return out

    def scale(self, alpha: float):
        check(lib.catgnn_model_scale(self.handle, alpha))

    def allreduce(self, comm: "Comm"):
        check(lib.catgnn_model_allreduce(self.handle, comm.handle))

    def close(self):
        if getattr(self, "handle", None):
            lib.catgnn_model_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def model_average(models: List[GNNModel], counts, dst: GNNModel):
    """train.cpp:154-172 over device-resident replicas (dst may be one of them)."""
    n = len(models)
    arr = (C.c_void_p * n)(*[m.handle.value for m in models])
    c = np.ascontiguousarray(counts, np.uint64)
    check(lib.catgnn_model_average(n, arr, _ptr(c), dst.handle))


def weighted_sum(models: List[GNNModel], alpha, dst: GNNModel):
    """dst = sum_i alpha_i models_i (model_average's loop with given weights):
    a rank's share of the cross-rank average, alpha from the global sync_weights."""
    n = len(models)
    arr = (C.c_void_p * n)(*[m.handle.value for m in models])
    a = np.ascontiguousarray(alpha, np.float64)
    check(lib.catgnn_model_weighted_sum(n, arr, _ptr(a), dst.handle))


class Comm:
    """NCCL communicator, one rank per GPU (C1)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib.catgnn_comm_unique_id(buf))
        return buf.raw

    def __init__(self, ctx: Context, nranks: int, rank: int, uid: bytes):
        h = C.c_void_p()
        buf = C.create_string_buffer(uid, 128)
        check(lib.catgnn_comm_create(ctx.handle, nranks, rank, buf, C.byref(h)))
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            lib.catgnn_comm_destroy(self.handle)
            self.handle = None


def sync_weights(counts):
    """train.cpp:139-152 (host arithmetic, bit-identical)."""
    total = int(sum(int(c) for c in counts))
    if len(counts) == 0 or total == 0:
        from ._lib import DataError
        raise DataError("model averaging requires a nonzero training-node count")
    alpha = [int(c) / total for c in counts[:-1]]
    alpha.append(1.0 - sum(alpha))
    return alpha


def assign_partitions(p: int, world: int, rank: int) -> List[int]:
    """Cyclic partition -> worker assignment (p % q == 0, train.cpp:293-294)."""
    if world == 0 or p == 0:
        from ._lib import ConfigError
        raise ConfigError("need at least one worker and one partition")
    if p % world:
        from ._lib import ConfigError
        raise ConfigError("partition count must be a multiple of the worker count")
    return list(range(rank, p, world))


@dataclass
class GNNTrainResult:
    params: np.ndarray
    losses: List[float] = field(default_factory=list)
    history: List[tuple] = field(default_factory=list)
    averaging_ops: int = 0


def distributed_train(kind, shards: List[Shard], counts, sync_interval: int, epochs: int, layers: int,
                      hidden: int, classes: int, seed: int = 0, optimizer=ADAM, lr: float = 0.01,
                      global_shard: Optional[Shard] = None, comm: Optional[Comm] = None,
                      alpha_all: Optional[List[float]] = None, want_loss: bool = True,
                      ctx: Optional[Context] = None) -> GNNTrainResult:
    """Train this rank's partitions (`shards`, with their global indices'
    train counts in `counts`) with averaging every `sync_interval` iterations.

    Single process: shards = all partitions, comm = None.  Multi-rank: each
    rank passes its own partitions and the NCCL comm; alpha_all is the full
    sync_weights vector restricted to this rank's partitions (same order)."""
    if sync_interval == 0:
        from ._lib import ConfigError
        raise ConfigError("sync interval must be >= 1")
    ctx = ctx or shards[0].ctx
    in_dim = shards[0].dim
    shared = GNNModel(kind, layers, in_dim, hidden, classes, optimizer, lr, seed, ctx=ctx)
    reps = [GNNModel(kind, layers, in_dim, hidden, classes, optimizer, lr, seed, ctx=ctx) for _ in shards]
    alpha = alpha_all if alpha_all is not None else sync_weights(counts)
    res = GNNTrainResult(params=None)
    done = 0
    while done < epochs:
        chunk = min(sync_interval, epochs - done)
        for r in reps:
            r.copy_params_from(shared)
        for _ in range(chunk):
            ep = 0.0
            for a, r, s in zip(alpha, reps, shards):
                l = r.train_step(s, want_loss)
                if want_loss:
                    ep += a * l
            res.losses.append(ep)
        if comm is None:
            model_average(reps, counts, shared)
        else:
            # C1: sum_i alpha_i theta_i over this rank's replicas with the global
            # alphas (a rank without train rows contributes zeros), then all-reduce
            weighted_sum(reps, alpha, shared)
            shared.allreduce(comm)
        done += chunk
        res.averaging_ops += 1
        if global_shard is not None:
            _, vf = shared.forward(global_shard, role=2) if global_shard.info.n_val else (None, 0.0)
            _, tf = shared.forward(global_shard, role=3) if global_shard.info.n_test else (None, 0.0)
            res.history.append((done, res.averaging_ops, vf, tf))
    res.params = shared.get_params()
    return res


def distributed_train_artifact(artifact_dir: str, kind, epochs: int, sync_interval: int, layers: int = 2,
                               hidden: int = 256, classes: int = 0, workers: int = 1, seed: int = 0,
                               optimizer=ADAM, lr: float = 0.01, beta1=0.9, beta2=0.999, eps=1e-8,
                               eval_global: bool = True, input: str = "", features: str = "",
                               comm: Optional[Comm] = None, ctx: Optional[Context] = None) -> GNNTrainResult:
    """catgnn_gnn_distributed_train: the whole loop in the library (C++ host
    side of the drop-in) on an artifact directory, like train-sim
    (proj/tools/gnnpart.cpp:310-321 -> distributed_train, train.cpp:289-340)."""
    ctx = ctx or default_context()
    k = KINDS[kind] if isinstance(kind, str) else kind
    cfg = GnnTrainConfig(ModelConfig(k, layers, 0, hidden, classes, optimizer, lr, beta1, beta2, eps, seed),
                         epochs, sync_interval, workers, int(eval_global))
    cap_h = epochs // max(sync_interval, 1) + 2
    he = np.zeros(cap_h, np.uint64); hs = np.zeros(cap_h, np.uint64)
    hv = np.zeros(cap_h); ht = np.zeros(cap_h)
    losses = np.zeros(max(epochs, 1))
    model = C.c_void_p()
    res = GnnResult(None, 0, 0, losses.ctypes.data, losses.size, 0, he.ctypes.data, hs.ctypes.data,
                    hv.ctypes.data, ht.ctypes.data, cap_h, 0, 0, 0, 0, C.cast(C.pointer(model), C.c_void_p))
    check(lib.catgnn_gnn_distributed_train(ctx.handle, str(artifact_dir).encode(), str(input).encode(),
                                           str(features).encode(), C.byref(cfg),
                                           comm.handle if comm else None, C.byref(res)))
    mc = ModelConfig(k, layers, res.in_dim, hidden, res.classes, optimizer, lr, beta1, beta2, eps, seed)
    m = GNNModel.adopt(model, ctx, mc)
    params = m.get_params()
    n = min(res.n_hist, cap_h)
    hist = [(int(he[i]), int(hs[i]), float(hv[i]), float(ht[i])) for i in range(n)]
    out = GNNTrainResult(params=params, losses=losses[:res.n_losses].tolist(), history=hist,
                         averaging_ops=int(res.averaging_ops))
    out.in_dim, out.classes = int(res.in_dim), int(res.classes)
    out.model = m
    return out
