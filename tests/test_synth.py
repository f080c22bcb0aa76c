"""The data formats either side of the path: RMAT generator invariants, the
NumPy 1-hop completion vs the reference's complete_edges + write_partitions,
and the upstream SPRING wrapper vs the reference partition pipeline."""
import os

import numpy as np
import pytest

from paper_2404_02300_b200 import synth

ROLE = {"none": 0, "train": 1, "val": 2, "test": 3}


def read_part(art, s):
    pd = os.path.join(art, f"part-{s}")
    raw = np.fromfile(os.path.join(pd, "edges.bin"), np.uint8)
    assert bytes(raw[:4]) == b"EDG1"
    edges = raw[4:].view(np.uint64).reshape(-1, 2)
    with open(os.path.join(pd, "nodes.tsv")) as f:
        rows = [ln.rstrip("\n").split("\t") for ln in f if ln.strip()]
    ext = np.array([int(r[0]) for r in rows], np.uint64)
    own = np.array([int(r[1]) for r in rows], np.uint8)
    role = np.array([ROLE[r[2]] for r in rows], np.uint8)
    return edges, ext, own, role


def test_rmat_invariants():
    e, n, seen = synth.rmat_edges(11, 8000, seed=5)
    assert e.shape == (8000, 2)
    assert np.all(e[:, 0] != e[:, 1])                      # no self-loops
    key = np.minimum(e[:, 0], e[:, 1]) * np.uint64(1 << 32) + np.maximum(e[:, 0], e[:, 1])
    assert np.unique(key).size == key.size                 # no duplicate unordered pairs
    assert set(np.unique(e).tolist()) == set(range(n))     # compact ids, all seen
    e2, n2, _ = synth.rmat_edges(11, 8000, seed=5)
    assert np.array_equal(e, e2) and n == n2               # deterministic


@pytest.mark.parametrize("scale,edges,seed", [(6, 200, 0), (9, 1500, 7), (12, 40000, 3), (14, 100000, 11)])
def test_cpp_generator_matches_numpy_statement(scale, edges, seed):
    a = synth.rmat_edges_numpy(scale, edges, seed=seed)
    b = synth.rmat_edges(scale, edges, seed=seed)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1]


def test_seed_for_matches_reference():
    from oracle import ref
    for s, k in [(0, 0), (1, 0xFEA7), (42, 7), (2**63 + 5, 2**40)]:
        assert synth.seed_for(s, k) == ref.seed_for(s, k)


@pytest.mark.parametrize("p", [1, 2, 4])
def test_completion_matches_reference_artifact(small_ds, p):
    from conftest import make_artifact
    from upstream.spring import spring_homes
    art = make_artifact(small_ds, p=p, with_features=False, tag="cmp")
    home, _ = spring_homes(small_ds["edge_file"], small_ds["n"], p)
    parts = synth.complete_edges(small_ds["edges"], home, small_ds["roles"], p)
    for s in range(p):
        edges, ext, own, role = read_part(art, s)
        assert np.array_equal(edges, parts[s].edges)
        assert np.array_equal(ext, parts[s].ext)
        assert np.array_equal(own, parts[s].owner)
        assert np.array_equal(role, parts[s].role)
    from oracle import ref
    rf, _ = ref.artifact_replication_factor(art)
    assert synth.replication_factor(parts, small_ds["n"]) == rf


def test_one_hop_closure(small_ds):
    # SPEC acceptance 5: every owner's in-partition degree equals its global degree
    from upstream.spring import spring_homes
    home, _ = spring_homes(small_ds["edge_file"], small_ds["n"], 4)
    parts = synth.complete_edges(small_ds["edges"], home, small_ds["roles"], 4)
    e = small_ds["edges"].astype(np.int64)
    gdeg = np.bincount(e.ravel(), minlength=small_ds["n"])
    for s, pt in enumerate(parts):
        ldeg = np.bincount(pt.edges.astype(np.int64).ravel(), minlength=small_ds["n"])
        owned = pt.ext[pt.owner == 1].astype(np.int64)
        assert np.array_equal(ldeg[owned], gdeg[owned])
