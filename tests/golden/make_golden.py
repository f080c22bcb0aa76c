"""Regenerates tests/golden/golden_small.npz from the UNMODIFIED reference
library (oracle/_ref/libgnnpart_ref.so, built from /root/reference/proj/src
with the Eigen shim).  Run from the repo root where /root/reference exists:

    python tests/golden/make_golden.py

The fixture holds a small RMAT dataset, the reference SPRING p=2 artifact
contents (per-partition edges and node tables, completion.cpp / store.cpp),
the reference CSR of every shard (build_adjacency, train.cpp:30-47), the
replication factor (metrics.cpp:9-12), sgc_propagate outputs (train.cpp:49-65),
a softmax_gradient (train.cpp:86-94), train_epochs params (train.cpp:96-128)
and a full distributed_train run (train.cpp:289-340).
"""
import os
import sys
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import ref  # noqa: E402
from paper_2404_02300_b200 import synth  # noqa: E402

SCALE, EDGES, DIM, CLASSES, SEED, P = 9, 1500, 8, 4, 7, 2
HOPS, EPOCHS, SYNC, LR, BATCH = 2, 6, 2, 0.05, 64


def main(out=os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden_small.npz")):
    e, n, _ = synth.rmat_edges(SCALE, EDGES, seed=SEED)
    lab, roles = synth.node_meta(n, CLASSES, 0.6, 0.2, 0.2, seed=SEED)
    X = synth.class_features(lab, DIM, CLASSES, seed=SEED)
    d = tempfile.mkdtemp()
    synth.write_dataset(d, e, lab, roles, X)
    art = os.path.join(d, "art")
    ref.partition(os.path.join(d, "edges.bin"), art, P, nodes=os.path.join(d, "nodes.tsv"),
                  features=os.path.join(d, "features.bin"))
    g = {"edges": e, "labels": lab, "roles": roles, "X": X, "num_nodes": np.int64(n)}
    rf, mrf = ref.artifact_replication_factor(art)
    g["rf"] = np.float64(rf)
    g["manifest_rf"] = np.float64(mrf)
    role_id = {"none": 0, "train": 1, "val": 2, "test": 3}
    for s in range(P):
        pd = os.path.join(art, f"part-{s}")
        raw = np.fromfile(os.path.join(pd, "edges.bin"), np.uint8)
        g[f"p{s}_edges"] = raw[4:].view(np.uint64).reshape(-1, 2)
        with open(os.path.join(pd, "nodes.tsv")) as f:
            rows = [ln.rstrip("\n").split("\t") for ln in f if ln.strip()]
        g[f"p{s}_ext"] = np.array([int(r[0]) for r in rows], np.uint64)
        g[f"p{s}_owner"] = np.array([int(r[1]) for r in rows], np.uint8)
        g[f"p{s}_role"] = np.array([role_id[r[2]] for r in rows], np.uint8)
    td = ref.TrainingData(art)
    for s in [-1] + list(range(P)):
        sh = td.shard(s)
        k = "g" if s < 0 else f"s{s}"
        g[f"{k}_offsets"] = sh.offsets
        g[f"{k}_neighbors"] = sh.neighbors
        g[f"{k}_labels"] = sh.labels
        g[f"{k}_train"] = sh.train_rows
        g[f"{k}_val"] = sh.val_rows
        g[f"{k}_test"] = sh.test_rows
        g[f"{k}_prop"] = ref.sgc_propagate(sh.offsets, sh.neighbors, sh.features, HOPS)
    # softmax_gradient on the first 50 train rows of shard 0 with a fixed W
    rng = np.random.default_rng(SEED)
    W0 = rng.normal(size=(DIM, CLASSES)) * 0.3
    b0 = rng.normal(size=CLASSES) * 0.1
    rows = g["s0_train"][:50]
    gW, gb = ref.softmax_gradient(W0, b0, g["s0_prop"][rows], g["s0_labels"][rows])
    g.update(W0=W0, b0=b0, grad_rows=rows, gW=gW, gb=gb,
             loss=np.float64(ref.softmax_loss(W0, b0, g["s0_prop"][rows], g["s0_labels"][rows])))
    W1, b1 = ref.train_epochs(np.zeros((DIM, CLASSES)), np.zeros(CLASSES), g["s0_prop"], g["s0_labels"],
                              g["s0_train"], LR, BATCH, 0, 3, 11)
    g.update(te_W=W1, te_b=b1)
    res = td.distributed_train(1, SYNC, epochs=EPOCHS, lr=LR, batch=BATCH, prop_hops=HOPS, seed=SEED)
    g.update(dt_W=res["W"], dt_b=res["b"], dt_hist=np.array(res["history"], np.float64),
             dt_ops=np.int64(res["averaging_ops"]))
    g["config"] = np.array([SCALE, EDGES, DIM, CLASSES, SEED, P, HOPS, EPOCHS, SYNC, BATCH], np.int64)
    g["lr"] = np.float64(LR)
    np.savez_compressed(out, **g)
    print("wrote", out, os.path.getsize(out), "bytes")


if __name__ == "__main__":
    main()
