"""B200-native CATGNN per-partition GNN training step (arxiv 2404.02300).

Drop-in for the reference's `gnnpart` training path (proj/src/train.cpp) behind
the C ABI in include/catgnn.h; see DESIGN.md.  Importing this package loads the
sm_100a library and fails loudly if it is missing (no CPU fallback).
"""
from . import gnnpart  # noqa: F401
from ._lib import LIB_PATH, ConfigError, DataError, InternalError  # noqa: F401

__version__ = "0.1.0"
