"""Shared fixtures.  `gpu`-marked tests need a B200 (run via gpurun); the rest run on CPU.

The oracle (oracle/_ref/libgnnpart_ref.so = the unmodified reference library)
is test infrastructure: it partitions synthetic graphs into real artifacts and
provides the reference outputs every parity test compares against.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: config-1 scale, tens of seconds")


def make_dataset(tmpdir, scale=10, edges=3000, dim=8, classes=4, seed=1, fracs=(0.7, 0.15, 0.15)):
    from paper_2404_02300_b200 import synth
    e, n, _ = synth.rmat_edges(scale, edges, seed=seed)
    lab, roles = synth.node_meta(n, classes, *fracs, seed=seed)
    X = synth.class_features(lab, dim, classes, seed=seed)
    d = os.path.join(str(tmpdir), f"data_s{scale}_e{edges}_d{dim}_c{classes}_r{seed}")
    synth.write_dataset(d, e, lab, roles, X)
    return dict(dir=d, edges=e, n=n, labels=lab, roles=roles, X=X,
                edge_file=os.path.join(d, "edges.bin"), nodes_file=os.path.join(d, "nodes.tsv"),
                feat_file=os.path.join(d, "features.bin"))


def make_artifact(ds, p=2, with_features=True, tag="art", **kw):
    from oracle import ref
    out = os.path.join(ds["dir"], f"{tag}_p{p}")
    if not os.path.exists(os.path.join(out, "manifest.json")):
        ref.partition(ds["edge_file"], out, p, nodes=ds["nodes_file"],
                      features=ds["feat_file"] if with_features else "", **kw)
    return out


@pytest.fixture(scope="session")
def small_ds(tmp_path_factory):
    return make_dataset(tmp_path_factory.mktemp("small"))


@pytest.fixture(scope="session")
def small_artifact(small_ds):
    return make_artifact(small_ds, p=2)


def rel_err(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    den = max(np.linalg.norm(b), 1e-30)
    return float(np.linalg.norm(a - b) / den)
