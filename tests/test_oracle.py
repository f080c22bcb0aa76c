"""Pins the CPU oracle (the unmodified reference library + Eigen shim) against
the reference's own known-answer vectors and the committed
golden fixture (tests/golden/golden_small.npz, made by make_golden.py)."""
import os

import numpy as np
import pytest

from oracle import ref

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "golden_small.npz")


def test_build_adjacency_kat():
    # build_adjacency(3, {(0,1),(0,2)}) -> offsets [0,2,3,4], neighbors [1,2,0,0]
    off, nb = ref.build_adjacency(3, np.array([[0, 1], [0, 2]]))
    assert off.tolist() == [0, 2, 3, 4]
    assert nb.tolist() == [1, 2, 0, 0]


def test_build_adjacency_multiset_and_loops():
    # duplicates stay, a self-loop is stored once (train.hpp:15-17)
    off, nb = ref.build_adjacency(3, np.array([[0, 1], [0, 1], [2, 2]]))
    assert off.tolist() == [0, 2, 4, 5]
    assert nb.tolist() == [1, 1, 0, 0, 2]


def test_build_adjacency_rejects_out_of_range():
    with pytest.raises(ref.RefError) as e:
        ref.build_adjacency(2, np.array([[0, 5]]))
    assert e.value.code == 3


def test_sgc_propagate_star_kat():
    # star centre 0, leaves 1,2; [[0],[3],[3]], k=1 -> 2, 1.5, 1.5
    off, nb = ref.build_adjacency(3, np.array([[0, 1], [0, 2]]))
    y = ref.sgc_propagate(off, nb, np.array([[0.0], [3.0], [3.0]]), 1)
    assert y.ravel().tolist() == [2.0, 1.5, 1.5]


def test_sgc_propagate_constants_and_identity():
    rng = np.random.default_rng(0)
    pairs = rng.integers(0, 20, size=(60, 2))
    off, nb = ref.build_adjacency(20, pairs)
    ones = np.ones((20, 3))
    np.testing.assert_allclose(ref.sgc_propagate(off, nb, ones, 3), ones, rtol=0, atol=1e-15)
    x = rng.normal(size=(20, 3))
    assert np.array_equal(ref.sgc_propagate(off, nb, x, 0), x)


def test_model_average_kats():
    # SPEC.md:491-493
    W, _ = ref.model_average(np.array([[[2.0]], [[4.0]]]), np.zeros((2, 1)), [1, 3])
    assert W[0, 0] == 3.5
    p = np.random.default_rng(1).normal(size=(3, 4, 2))
    same = np.stack([p[0]] * 3)
    W, _ = ref.model_average(same, np.zeros((3, 2)), [5, 1, 2])
    np.testing.assert_allclose(W, p[0], rtol=1e-15)
    W, _ = ref.model_average(p[:2], np.zeros((2, 2)), [7, 0])
    np.testing.assert_array_equal(W, p[0])
    with pytest.raises(ref.RefError) as e:
        ref.model_average(p[:2], np.zeros((2, 2)), [0, 0])
    assert e.value.code == 3


def test_sync_weights_last_absorbs_rounding():
    a = ref.sync_weights([1, 1, 1])
    assert a.sum() == 1.0 and a[2] == 1.0 - (a[0] + a[1])


def test_micro_f1_kats():
    # all correct -> 1.0; constant predictor on balanced 4-class data -> 0.25
    x = np.eye(4)
    W = np.eye(4) * 5
    assert ref.evaluate_micro_f1(W, np.zeros(4), x, np.arange(4), np.arange(4)) == 1.0
    Wc = np.zeros((4, 4))
    bc = np.array([0, 0, 1.0, 0])
    assert ref.evaluate_micro_f1(Wc, bc, x, np.arange(4), np.arange(4)) == 0.25
    with pytest.raises(ref.RefError):
        ref.evaluate_micro_f1(W, np.zeros(4), x, np.arange(4), np.array([], np.uint32))


def test_gradient_check_central_differences():
    # SPEC acceptance 10: analytic vs central differences, rel err < 1e-4 on 20 instances
    rng = np.random.default_rng(2)
    for _ in range(20):
        d, c, n = rng.integers(2, 6), rng.integers(2, 5), rng.integers(3, 9)
        W = rng.normal(size=(d, c)); b = rng.normal(size=c)
        x = rng.normal(size=(n, d)); y = rng.integers(0, c, n)
        gW, _ = ref.softmax_gradient(W, b, x, y)
        num = np.zeros_like(W)
        for i in range(d):
            for j in range(c):
                Wp = W.copy(); Wp[i, j] += 1e-6
                Wm = W.copy(); Wm[i, j] -= 1e-6
                num[i, j] = (ref.softmax_loss(Wp, b, x, y) - ref.softmax_loss(Wm, b, x, y)) / 2e-6
        assert np.abs(num - gW).max() / max(np.abs(gW).max(), 1e-12) < 1e-4


def test_train_epochs_lr0_and_determinism():
    rng = np.random.default_rng(3)
    x = rng.normal(size=(40, 5)); y = rng.integers(0, 3, 40)
    tr = np.arange(0, 40, 2, dtype=np.uint32)
    W0 = rng.normal(size=(5, 3)); b0 = rng.normal(size=3)
    W, b = ref.train_epochs(W0, b0, x, y, tr, 0.0, 8, 0, 4, 9)
    assert np.array_equal(W, W0) and np.array_equal(b, b0)
    Wa, ba = ref.train_epochs(W0, b0, x, y, tr, 0.1, 8, 0, 4, 9)
    Wb, bb = ref.train_epochs(W0, b0, x, y, tr, 0.1, 8, 0, 4, 9)
    assert np.array_equal(Wa, Wb) and np.array_equal(ba, bb)


def test_oracle_reproduces_golden(tmp_path):
    """The oracle rebuilt here must reproduce the committed reference outputs exactly."""
    from paper_2404_02300_b200 import synth
    g = np.load(GOLDEN)
    scale, edges, dim, classes, seed, p, hops, epochs, sync, batch = g["config"].tolist()
    e, n, _ = synth.rmat_edges(scale, edges, seed=seed)
    assert np.array_equal(e, g["edges"]) and n == int(g["num_nodes"])
    lab, roles = synth.node_meta(n, classes, 0.6, 0.2, 0.2, seed=seed)
    X = synth.class_features(lab, dim, classes, seed=seed)
    assert np.array_equal(X, g["X"])
    synth.write_dataset(str(tmp_path), e, lab, roles, X)
    art = str(tmp_path / "art")
    ref.partition(str(tmp_path / "edges.bin"), art, p, nodes=str(tmp_path / "nodes.tsv"),
                  features=str(tmp_path / "features.bin"))
    rf, mrf = ref.artifact_replication_factor(art)
    assert rf == g["rf"] and mrf == g["manifest_rf"]
    td = ref.TrainingData(art)
    for s in [-1] + list(range(p)):
        k = "g" if s < 0 else f"s{s}"
        sh = td.shard(s)
        assert np.array_equal(sh.offsets, g[f"{k}_offsets"])
        assert np.array_equal(sh.neighbors, g[f"{k}_neighbors"])
        assert np.array_equal(ref.sgc_propagate(sh.offsets, sh.neighbors, sh.features, hops), g[f"{k}_prop"])
    res = td.distributed_train(1, sync, epochs=epochs, lr=float(g["lr"]), batch=batch, prop_hops=hops, seed=seed)
    assert np.array_equal(res["W"], g["dt_W"])
    assert np.array_equal(np.array(res["history"], np.float64), g["dt_hist"])


def test_distributed_independent_of_worker_count(small_artifact):
    # train.hpp:118-122: results do not depend on q
    td = ref.TrainingData(small_artifact)
    a = td.distributed_train(1, 2, epochs=4, batch=64)
    b = td.distributed_train(2, 2, epochs=4, batch=64)
    assert np.array_equal(a["W"], b["W"]) and a["history"] == b["history"]
    with pytest.raises(ref.RefError) as e:
        td.distributed_train(3, 2, epochs=4)
    assert e.value.code == 2
