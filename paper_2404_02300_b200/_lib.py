"""ctypes binding of libcatgnn.so (include/catgnn.h).

The product path has no CPU fallback: if the CUDA library is missing this
module raises at import time with the build command to run.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# CATGNN_LIB: an alternative in-tree build of the same library (kernel A/B runs)
LIB_PATH = os.environ.get("CATGNN_LIB") or os.path.join(_HERE, "libcatgnn.so")


class CatgnnError(RuntimeError):
    code = 4


class ConfigError(CatgnnError):
    """Reference ConfigError (proj/include/gnnpart/common.hpp:17-19), CLI exit 2."""
    code = 2


class DataError(CatgnnError):
    """Reference DataError (proj/include/gnnpart/common.hpp:21-24), CLI exit 3."""
    code = 3


class InternalError(CatgnnError):
    code = 4


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libcatgnn.so not built ({LIB_PATH}); run `make -C {_HERE}` or "
            "`python -c 'import __graft_entry__ as g; g.build()'` — there is no CPU fallback")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, u32, u64, i32, f64 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int32, C.c_double
    P = C.POINTER
    sig = {
        "catgnn_last_error": (C.c_char_p, []),
        "catgnn_version": (C.c_int, []),
        "catgnn_ctx_create": (C.c_int, [C.c_int, vp, P(vp)]),
        "catgnn_ctx_destroy": (C.c_int, [vp]),
        "catgnn_ctx_synchronize": (C.c_int, [vp]),
        "catgnn_ctx_launch_count": (u64, [vp]),
        "catgnn_ctx_set_kernel_timing": (C.c_int, [vp, C.c_int]),
        "catgnn_ctx_wait": (C.c_int, [vp, vp]),
        "catgnn_features_reset_deps": (C.c_int, [vp]),
        "catgnn_split_features": (C.c_int, [vp, vp, C.c_char_p, C.c_char_p, P(u32)]),
        "catgnn_model_last_loss_async": (C.c_int, [vp, P(f64), P(u64)]),
        "catgnn_ctx_set_sm_budget": (C.c_int, [vp, C.c_int, C.c_int]),
        "catgnn_ctx_kernel_time": (C.c_int, [vp, P(f64), P(u64), P(f64), P(u64)]),
        "catgnn_ctx_timing_record": (C.c_int, [vp, u32, C.c_char_p, u32, P(u32)]),
        "catgnn_artifact_open": (C.c_int, [C.c_char_p, P(vp)]),
        "catgnn_artifact_close": (C.c_int, [vp]),
        "catgnn_artifact_get_info": (C.c_int, [vp, vp]),
        "catgnn_artifact_part_counts": (C.c_int, [vp, u32, P(u64), P(u64), P(u64)]),
        "catgnn_artifact_replica_map": (C.c_int, [vp, u32, vp, vp, vp, vp]),
        "catgnn_shard_halo_map": (C.c_int, [vp, vp, vp, vp]),
        "catgnn_shard_train_views": (C.c_int, [vp, vp, vp, vp]),
        "catgnn_shard_load": (C.c_int, [vp, vp, i32, C.c_char_p, C.c_char_p, P(vp)]),
        "catgnn_shard_create": (C.c_int, [vp, u32, vp, u64, vp, u32, P(vp)]),
        "catgnn_shard_create_from_part": (C.c_int, [vp, u64, vp, vp, vp, vp, vp, u64, vp, u32, P(vp)]),
        "catgnn_shard_destroy": (C.c_int, [vp]),
        "catgnn_shard_set_labels": (C.c_int, [vp, vp, vp, u64, vp, u64, vp, u64]),
        "catgnn_shard_upload_features": (C.c_int, [vp, vp, u32]),
        "catgnn_features_create": (C.c_int, [vp, u64, u32, P(vp)]),
        "catgnn_features_destroy": (C.c_int, [vp]),
        "catgnn_features_upload": (C.c_int, [vp, vp, u64, u64]),
        "catgnn_shard_gather_features": (C.c_int, [vp, vp]),
        "catgnn_shard_set_feature_layout": (C.c_int, [vp, C.c_int]),
        "catgnn_features_allgather": (C.c_int, [vp, vp, u64]),
        "catgnn_complete_edges": (C.c_int, [vp, vp, u64, vp, vp, u64, u32, u32, P(vp)]),
        "catgnn_complete_edges_indexed": (C.c_int, [vp, vp, vp, u64, vp, vp, u32, u32, P(vp)]),
        "catgnn_complete_edges_file": (C.c_int, [vp, C.c_char_p, C.c_int, vp, vp, u64, u32, u32, P(vp)]),
        "catgnn_index_build": (C.c_int, [vp, vp, u64, P(vp)]),
        "catgnn_index_info": (C.c_int, [vp, P(u64), P(u64), P(u64)]),
        "catgnn_index_export": (C.c_int, [vp, vp, vp]),
        "catgnn_index_destroy": (C.c_int, [vp]),
        "catgnn_completion_part_counts": (C.c_int, [vp, u32, P(u64), P(u64), P(u64)]),
        "catgnn_completion_part": (C.c_int, [vp, u32, vp, vp, vp, vp]),
        "catgnn_completion_destroy": (C.c_int, [vp]),
        "catgnn_probe_read_bandwidth": (C.c_int, [vp, u64, C.c_int, P(f64)]),
        "catgnn_shard_get_info": (C.c_int, [vp, vp]),
        "catgnn_csr_export": (C.c_int, [vp, vp, vp]),
        "catgnn_shard_role_rows": (C.c_int, [vp, C.c_int, vp]),
        "catgnn_shard_labels": (C.c_int, [vp, vp]),
        "catgnn_shard_export_features": (C.c_int, [vp, C.c_int, vp]),
        "catgnn_sgc_propagate": (C.c_int, [vp, u32]),
        "catgnn_softmax_loss": (C.c_int, [vp, vp, vp, u32, vp, u64, P(f64)]),
        "catgnn_softmax_gradient": (C.c_int, [vp, vp, vp, u32, vp, u64, vp, vp]),
        "catgnn_train_epochs": (C.c_int, [u32, vp, vp, vp, u32, f64, u32, u64, u64, vp]),
        "catgnn_sync_weights": (C.c_int, [vp, u32, vp]),
        "catgnn_model_average_host": (C.c_int, [vp, u32, vp, u64, vp, vp]),
        "catgnn_evaluate_micro_f1": (C.c_int, [vp, vp, vp, u32, vp, u64, P(f64)]),
        "catgnn_distributed_train": (C.c_int, [u32, vp, vp, u32, u32, vp, vp]),
        "catgnn_model_create": (C.c_int, [vp, vp, P(vp)]),
        "catgnn_model_destroy": (C.c_int, [vp]),
        "catgnn_model_set_act_f16": (C.c_int, [vp, C.c_int]),
        "catgnn_model_num_params": (u64, [vp]),
        "catgnn_model_layer_shape": (C.c_int, [vp, u32, P(u32), P(u32), P(u64), P(u64)]),
        "catgnn_model_get_params": (C.c_int, [vp, vp]),
        "catgnn_model_set_params": (C.c_int, [vp, vp]),
        "catgnn_model_copy_params": (C.c_int, [vp, vp]),
        "catgnn_model_get_grads": (C.c_int, [vp, vp]),
        "catgnn_model_train_step": (C.c_int, [vp, vp, P(f64)]),
        "catgnn_model_last_loss": (C.c_int, [vp, P(f64)]),
        "catgnn_model_forward_backward": (C.c_int, [vp, vp, P(f64)]),
        "catgnn_model_forward": (C.c_int, [vp, vp, vp, C.c_int, P(f64)]),
        "catgnn_model_export": (C.c_int, [vp, u32, C.c_int, vp, P(u32)]),
        "catgnn_model_average": (C.c_int, [u32, vp, vp, vp]),
        "catgnn_model_weighted_sum": (C.c_int, [u32, vp, vp, vp]),
        "catgnn_gnn_distributed_train": (C.c_int, [vp, C.c_char_p, C.c_char_p, C.c_char_p, vp, vp, vp]),
        "catgnn_train_local": (C.c_int, [vp, vp, vp, vp, P(u32)]),
        "catgnn_comm_unique_id": (C.c_int, [vp]),
        "catgnn_comm_create": (C.c_int, [vp, C.c_int, C.c_int, vp, P(vp)]),
        "catgnn_comm_destroy": (C.c_int, [vp]),
        "catgnn_model_scale": (C.c_int, [vp, f64]),
        "catgnn_model_allreduce": (C.c_int, [vp, vp]),
        "catgnn_gemm_tn": (C.c_int, [vp, u32, u32, u32, vp, vp, vp, u32, C.c_int]),
        "catgnn_gemm": (C.c_int, [vp, u32, u32, u32, vp, C.c_int, vp, C.c_int, vp, u32, C.c_int]),
        "catgnn_synth_rmat": (C.c_int, [u32, u64, f64, f64, f64, u64, vp, P(u64)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()

EXPORTED = [
    "catgnn_last_error", "catgnn_version", "catgnn_ctx_create", "catgnn_ctx_destroy",
]


def check(rc: int):
    if rc == 0:
        return
    msg = lib.catgnn_last_error().decode(errors="replace")
    cls = {2: ConfigError, 3: DataError}.get(rc, InternalError)
    raise cls(msg)


class ArtifactInfo(C.Structure):
    _fields_ = [("num_partitions", C.c_uint32), ("num_nodes", C.c_uint64), ("num_edges", C.c_uint64),
                ("feature_dim", C.c_uint32), ("has_features", C.c_int), ("has_meta", C.c_int),
                ("add_reverse", C.c_int), ("replication_factor", C.c_double),
                ("manifest_replication_factor", C.c_double)]


class ShardInfo(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("nnz", C.c_uint64), ("dim", C.c_uint32), ("classes", C.c_uint32),
                ("n_train", C.c_uint64), ("n_val", C.c_uint64), ("n_test", C.c_uint64),
                ("heavy_rows", C.c_uint64), ("tasks", C.c_uint64)]


class TrainConfig(C.Structure):
    """TrainConfig (proj/include/gnnpart/train.hpp:42-48)."""
    _fields_ = [("epochs", C.c_uint32), ("lr", C.c_double), ("batch", C.c_uint32),
                ("prop_hops", C.c_uint32), ("seed", C.c_uint64)]

    def __init__(self, epochs=100, lr=0.01, batch=512, prop_hops=2, seed=0):
        super().__init__(epochs, lr, batch, prop_hops, seed)


class DistResult(C.Structure):
    _fields_ = [("W", C.c_void_p), ("b", C.c_void_p), ("dim", C.c_uint32), ("classes", C.c_uint32),
                ("hist_epoch", C.c_void_p), ("hist_syncs", C.c_void_p), ("hist_val", C.c_void_p),
                ("hist_test", C.c_void_p), ("hist_capacity", C.c_uint64), ("n_hist", C.c_uint64),
                ("averaging_ops", C.c_uint64)]


class ModelConfig(C.Structure):
    _fields_ = [("kind", C.c_int), ("layers", C.c_uint32), ("in_dim", C.c_uint32), ("hidden", C.c_uint32),
                ("classes", C.c_uint32), ("optimizer", C.c_int), ("lr", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("seed", C.c_uint64)]


class GnnTrainConfig(C.Structure):
    _fields_ = [("model", ModelConfig), ("epochs", C.c_uint32), ("sync_interval", C.c_uint32),
                ("workers", C.c_uint32), ("eval_global", C.c_int)]


class GnnResult(C.Structure):
    _fields_ = [("params", C.c_void_p), ("params_capacity", C.c_uint64), ("num_params", C.c_uint64),
                ("losses", C.c_void_p), ("loss_capacity", C.c_uint64), ("n_losses", C.c_uint64),
                ("hist_epoch", C.c_void_p), ("hist_syncs", C.c_void_p), ("hist_val", C.c_void_p),
                ("hist_test", C.c_void_p), ("hist_capacity", C.c_uint64), ("n_hist", C.c_uint64),
                ("averaging_ops", C.c_uint64), ("in_dim", C.c_uint32), ("classes", C.c_uint32),
                ("model_out", C.c_void_p)]
