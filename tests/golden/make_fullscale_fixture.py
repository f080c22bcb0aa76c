"""Freezes the float64 oracle's 10-epoch run of a bench workload (BASELINE
configs[1]: reddit_gcn) into tests/golden/fullscale_<workload>.json — the
per-epoch loss (sum_i alpha_i mean-CE_i) and the averaged
model's test accuracy on the global graph — so the -m gpu suite can check the
north-star acceptance (loss within 1e-3 relative over the first 10 epochs, final
accuracy within 0.5 pt) at full size without re-running the oracle
(tests/test_gpu_fullscale.py::test_ten_epochs_match_frozen_oracle).

CPU only (no GPU needed): the workload is prepared with the NumPy completion and
the oracle runs in one process per partition.

    python tests/golden/make_fullscale_fixture.py [WORKLOAD] [EPOCHS]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
WORKLOAD = sys.argv[1] if len(sys.argv) > 1 else "reddit_gcn"
EPOCHS = int(sys.argv[2]) if len(sys.argv) > 2 else 10
import fullscale_ten_epochs as F  # noqa: E402

if __name__ == "__main__":
    o = F.run_oracle(EPOCHS, WORKLOAD)
    out = dict(workload=WORKLOAD, workload_key=o["key"], epochs=EPOCHS, seed=F.SEED, hidden=F.HIDDEN, lr=F.LR,
               sync_interval=1, optimizer="adam", losses=o["losses"], test_acc=o["test_acc"],
               test_rows=o["test_rows"], train_counts=o["counts"],
               num_nodes=o["meta"]["num_nodes"], part_rows=o["meta"]["part_rows"],
               part_edges=o["meta"]["part_edges"], oracle_seconds=o["seconds"],
               generator="tests/golden/make_fullscale_fixture.py (oracle/gnn_oracle.py, float64)")
    path = os.path.join(ROOT, "tests", "golden", f"fullscale_{WORKLOAD}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "part_rows"}))
