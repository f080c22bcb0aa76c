"""SGC path at shapes past one CTA's shared memory (sgc.cu): the
reference accepts any dim x classes and any batch (train.cpp:86-128), so the
device must too.  Each case is compared with the compiled reference
(oracle/_ref) on the same propagated features:

* the reference's default batch 512 with papers-like 128-d features and 172
  classes (dim*C + batch*C = 441 KB of parameters + probabilities);
* softmax_gradient over a whole train set at reddit width (602 x 41,
  batch = rows = 3000);
* more than 256 classes (softmax_loss / evaluate_micro_f1 / train_epochs)."""
import numpy as np
import pytest

from conftest import rel_err
from oracle import ref

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gp():
    from paper_2404_02300_b200 import gnnpart
    return gnnpart


def shard(gp, rows, dim, classes, seed):
    rng = np.random.default_rng(seed)
    pairs = rng.integers(0, rows, size=(rows * 4, 2)).astype(np.uint32)
    x = rng.normal(size=(rows, dim)).astype(np.float32)
    labels = rng.integers(0, classes, rows).astype(np.int32)
    labels[0] = classes - 1  # classes = max(label) + 1
    s = gp.Shard.from_edges(rows, pairs, x)
    s.set_labels(labels)
    xp = gp.sgc_propagate(s, 1)
    return s, xp.astype(np.float64), labels


def test_train_epochs_papers_width_default_batch(gp):
    rows, dim, C = 1500, 128, 172
    s, xp, labels = shard(gp, rows, dim, C, 1)
    train = np.sort(np.random.default_rng(2).choice(rows, 1100, replace=False)).astype(np.uint32)
    s.set_labels(labels, train)
    P = gp.zero_params(dim, C)
    gp.train_epochs(P, s, gp.TrainConfig(lr=0.05, batch=512), 0, 2, 7)
    W, b = ref.train_epochs(np.zeros((dim, C)), np.zeros(C), xp, labels, train, 0.05, 512, 0, 2, 7)
    assert rel_err(P.weight, W) < 1e-4 and rel_err(P.bias, b) < 1e-4


def test_softmax_gradient_whole_train_set_reddit_width(gp):
    rows, dim, C = 3000, 602, 41
    s, xp, labels = shard(gp, rows, dim, C, 3)
    rng = np.random.default_rng(4)
    P = gp.ModelParams((rng.normal(size=(dim, C)) * 0.05).astype(np.float32),
                       (rng.normal(size=C) * 0.1).astype(np.float32))
    r = np.arange(rows, dtype=np.uint32)
    gW, gb = gp.softmax_gradient(P, s, r)
    rW, rb = ref.softmax_gradient(P.weight.astype(np.float64), P.bias.astype(np.float64), xp, labels)
    assert rel_err(gW, rW) < 1e-4 and rel_err(gb, rb) < 1e-4


def test_more_than_256_classes(gp):
    rows, dim, C = 900, 24, 300
    s, xp, labels = shard(gp, rows, dim, C, 5)
    rng = np.random.default_rng(6)
    P = gp.ModelParams((rng.normal(size=(dim, C)) * 0.3).astype(np.float32),
                       (rng.normal(size=C) * 0.1).astype(np.float32))
    Wd, bd = P.weight.astype(np.float64), P.bias.astype(np.float64)
    r = np.arange(rows, dtype=np.uint32)
    assert abs(gp.softmax_loss(P, s, r) - ref.softmax_loss(Wd, bd, xp, labels)) < 1e-5 * ref.softmax_loss(
        Wd, bd, xp, labels)
    f1 = gp.evaluate_micro_f1(P, s, r)
    rf1 = ref.evaluate_micro_f1(Wd, bd, xp, labels, r)
    assert abs(f1 - rf1) <= 1.0 / rows + 1e-12
    s.set_labels(labels, r)
    Q = gp.zero_params(dim, C)
    gp.train_epochs(Q, s, gp.TrainConfig(lr=0.1, batch=64), 0, 2, 3)
    W, b = ref.train_epochs(np.zeros((dim, C)), np.zeros(C), xp, labels, r, 0.1, 64, 0, 2, 3)
    assert rel_err(Q.weight, W) < 1e-4 and rel_err(Q.bias, b) < 1e-4
