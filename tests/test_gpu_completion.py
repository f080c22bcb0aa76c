"""GPU neighbour completion (csrc/completion.cu) against the reference's own
complete_edges + write_partitions (oracle/_ref, the unmodified
proj/src/completion.cpp): bit-exact edges (first occurrence per unordered pair,
original orientation, stream order), node tables, owner flags and roles, for
1/2/3 hops on streams with duplicate and reversed records."""
import os

import numpy as np
import pytest

from oracle import ref
from test_synth import read_part

pytestmark = pytest.mark.gpu


def dup_stream(tmp, scale, edges, seed, classes=4):
    from paper_2404_02300_b200 import synth
    e, n, _ = synth.rmat_edges(scale, edges, seed=seed)
    rng = np.random.default_rng(seed)
    extra = e[rng.choice(e.shape[0], e.shape[0] // 5, replace=False)].copy()
    flip = rng.random(extra.shape[0]) < 0.5
    extra[flip] = extra[flip][:, ::-1]                 # reversed duplicates
    stream = np.concatenate([e, extra])
    stream = stream[rng.permutation(stream.shape[0])]  # duplicates before/after originals
    lab, roles = synth.node_meta(n, classes, 0.6, 0.2, 0.2, seed=seed)
    X = synth.class_features(lab, 4, classes, seed=seed)
    d = os.path.join(str(tmp), f"dup_{scale}_{edges}_{seed}")
    synth.write_dataset(d, stream, lab, roles, X)
    return dict(dir=d, edges=stream, n=n, roles=roles, edge_file=os.path.join(d, "edges.bin"),
                nodes_file=os.path.join(d, "nodes.tsv"))


@pytest.mark.parametrize("p,hops,scale,edges,seed", [(2, 1, 10, 3000, 1), (4, 1, 12, 20000, 2),
                                                     (8, 1, 12, 30000, 3), (4, 2, 11, 6000, 4),
                                                     (3, 3, 10, 2500, 5), (1, 1, 9, 800, 6)])
def test_device_completion_matches_reference(tmp_path, p, hops, scale, edges, seed):
    from paper_2404_02300_b200 import gnnpart as gp
    ds = dup_stream(tmp_path, scale, edges, seed)
    art = os.path.join(ds["dir"], f"art_p{p}_h{hops}")
    ref.partition(ds["edge_file"], art, p, nodes=ds["nodes_file"], hops=hops)
    ref_parts = [read_part(art, s) for s in range(p)]
    home = np.full(ds["n"], p, np.uint32)
    for s, (_, ext, own, _) in enumerate(ref_parts):
        home[ext[own == 1].astype(np.int64)] = s
    assert np.all(home < p)
    parts = gp.complete_edges(ds["edges"], home, ds["roles"], p, hops=hops)
    for s in range(p):
        edges, ext, own, role = ref_parts[s]
        assert np.array_equal(parts[s].edges, edges), s
        assert np.array_equal(parts[s].ext, ext), s
        assert np.array_equal(parts[s].owner, own), s
        assert np.array_equal(parts[s].role, role), s
    rf, _ = ref.artifact_replication_factor(art)
    assert sum(pt.rows for pt in parts) / ds["n"] == rf


def test_device_completion_errors():
    from paper_2404_02300_b200 import gnnpart as gp
    e = np.array([[0, 1], [1, 2]], np.uint64)
    with pytest.raises(gp.ConfigError, match="hop count"):
        gp.complete_edges(e, np.zeros(3, np.uint32), None, 1, hops=4)
    with pytest.raises(gp.DataError, match="home partition out of range"):
        gp.complete_edges(e, np.array([0, 1, 2], np.uint32), None, 2)
    with pytest.raises(gp.DataError, match="dense"):
        gp.complete_edges(np.array([[0, 5]], np.uint64), np.zeros(3, np.uint32), None, 1)
    # isolated owned node: present in its home's table without edges (completion.cpp:37)
    parts = gp.complete_edges(e, np.array([0, 0, 0, 1], np.uint32), None, 2)
    assert parts[1].ext.tolist() == [3] and parts[1].owner.tolist() == [1] and parts[1].edges.shape == (0, 2)


def sparse_id_stream(rng, n, m, self_loops=True):
    """Records over arbitrary 64-bit external ids (not dense, not sorted)."""
    ids = rng.choice(np.uint64(1) << np.uint64(62), size=n, replace=False).astype(np.uint64)
    a = rng.integers(0, n, size=m)
    b = rng.integers(0, n, size=m)
    if not self_loops:
        b = np.where(a == b, (b + 1) % n, b)
    return ids, np.stack([ids[a], ids[b]], 1).astype(np.uint64)


@pytest.mark.parametrize("n,m,seed", [(1, 1, 0), (50, 200, 1), (3000, 20000, 2), (40000, 300000, 3)])
def test_device_compute_degrees_matches_reference(tmp_path, n, m, seed):
    """compute_degrees (edge_stream.cpp:192-215): first-seen interning order,
    degrees with self-loops counting 2, record and self-loop counts."""
    from paper_2404_02300_b200 import gnnpart as gp
    rng = np.random.default_rng(seed)
    _, e = sparse_id_stream(rng, n, m)
    f = os.path.join(str(tmp_path), "edges.bin")
    with open(f, "wb") as fh:
        fh.write(b"EDG1")
        e.tofile(fh)
    d2e, deg, rm, rsl = ref.compute_degrees(f, 2 * m)
    idx = gp.compute_degrees(e)
    assert np.array_equal(idx.dense_to_ext, d2e)
    assert np.array_equal(idx.degree, deg)
    assert (idx.num_edges, idx.num_self_loops) == (rm, rsl)


@pytest.mark.parametrize("p,hops", [(2, 1), (4, 1), (3, 2)])
def test_indexed_completion_matches_reference(tmp_path, p, hops):
    """complete_edges over arbitrary 64-bit ids through the device index, vs the
    reference pipeline (compute_degrees -> SPRING -> complete_edges ->
    write_partitions) on the same EDG1 stream."""
    from paper_2404_02300_b200 import gnnpart as gp
    rng = np.random.default_rng(10 + p + hops)
    _, e = sparse_id_stream(rng, 2500, 12000, self_loops=False)
    e = np.concatenate([e, e[:1500, ::-1]])  # reversed duplicates
    d = str(tmp_path)
    f = os.path.join(d, "edges.bin")
    with open(f, "wb") as fh:
        fh.write(b"EDG1")
        e.tofile(fh)
    art = os.path.join(d, f"art_{p}_{hops}")
    ref.partition(f, art, p, hops=hops)
    ref_parts = [read_part(art, s) for s in range(p)]
    idx = gp.compute_degrees(e)
    dense_of = {int(x): i for i, x in enumerate(idx.dense_to_ext)}
    home = np.full(idx.num_nodes, p, np.uint32)
    for s, (_, ext, own, _) in enumerate(ref_parts):
        for x in ext[own == 1]:
            home[dense_of[int(x)]] = s
    assert np.all(home < p)
    parts = gp.complete_edges(e, home, None, p, hops=hops, index=idx)
    for s in range(p):
        edges, ext, own, role = ref_parts[s]
        assert np.array_equal(parts[s].edges, edges), s
        assert np.array_equal(parts[s].ext, ext), s
        assert np.array_equal(parts[s].owner, own), s
        assert np.array_equal(parts[s].role, role), s


@pytest.mark.parametrize("p,hops,add_reverse", [(4, 1, False), (3, 2, True), (2, 1, True)])
def test_streamed_file_completion_matches_in_memory(tmp_path, p, hops, add_reverse):
    """catgnn_complete_edges_file (EDG1 streamed through a pinned chunk, add_reverse
    expanded on the device) equals the in-memory path on the reference reader's
    stream (duplicates, reversed records, self-loops; 7-record chunks)."""
    from paper_2404_02300_b200 import gnnpart as gp
    os.environ["CATGNN_STREAM_CHUNK"] = "7"
    ds = dup_stream(tmp_path, 10, 3000, 11 + p)
    e = ds["edges"].copy()
    e[:40, 1] = e[:40, 0]  # self-loops (add_reverse keeps them single)
    path = os.path.join(str(tmp_path), "loops.bin")
    _write_edg1(path, e)
    rng = np.random.default_rng(p)
    home = rng.integers(0, p, ds["n"]).astype(np.uint32)
    want_stream = e if not add_reverse else np.concatenate(
        [np.stack([r, r[::-1]]) if r[0] != r[1] else r[None] for r in e]).reshape(-1, 2)
    want = gp.complete_edges(want_stream, home, ds["roles"], p, hops)
    got = gp.complete_edges_file(path, home, ds["roles"], p, hops, add_reverse=add_reverse)
    for a, b in zip(want, got):
        assert np.array_equal(a.edges, b.edges) and np.array_equal(a.ext, b.ext)
        assert np.array_equal(a.owner, b.owner) and np.array_equal(a.role, b.role)


def _write_edg1(path, e):
    with open(path, "wb") as f:
        f.write(b"EDG1")
        f.write(np.ascontiguousarray(e, np.uint64).tobytes())
