"""Validates bench.py's CPU-baseline extrapolation: the
reference's sgc_propagate (oracle/_ref, compiled unmodified) over ONE WHOLE
partition of the bench workload, one pass per width, on one core — against the
rate bench.py's bounded samples (self-contained row-block subgraphs) predict
for the same partition and widths, also on one core.

    python scripts/ref_full_pass.py [WORKLOAD] [PART] [WIDTHS]   (default reddit_gcn 0 41,256)

Writes one JSON line to stdout and gpurun_out/ref_full_pass.json.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    workload = sys.argv[1] if len(sys.argv) > 1 else "reddit_gcn"
    part = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    widths = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "41,256").split(",")]
    import bench
    from oracle import ref
    from benchdata import workloads as W
    w = W.WORKLOADS[workload]
    prep = W.prepare(w, lambda *a: None, native=False)
    d = prep["dir"]
    edges = np.load(os.path.join(d, f"p{part}_edges.npy"))
    ext = np.load(os.path.join(d, f"p{part}_ext.npy"))
    local = np.searchsorted(ext, edges.ravel()).astype(np.uint32).reshape(-1, 2)
    off, nb = ref.build_adjacency(ext.size, local)
    rows, nnz = ext.size, int(off[-1])
    full = {}
    for wd in widths:
        x = np.random.default_rng(wd).standard_normal(rows * wd)
        t0 = time.perf_counter()
        ref.sgc_propagate_colmajor(off, nb, x, rows, wd, 1)
        full[wd] = nnz / (time.perf_counter() - t0)
    # bench.py's estimate: self-contained samples of ~300k edges on one core
    # (cpu_reference_rate with one job at a time: raw and gather-source-corrected)
    nblk = 4
    jobs = bench.reference_jobs(prep, [(part, b * 17) for b in range(nblk)], 300_000)

    class One:  # this partition's schedule restricted to one width
        def __init__(self, wd):
            self.wd = wd

        def passes(self):
            return [self.wd]
    est, raw = {}, {}
    for wd in widths:
        es = tc = tr = 0.0
        for jb in jobs:
            rate, _, sample = bench.cpu_reference_rate(One(wd), [jb])
            e = jb[3]
            es += e
            tc += e / rate
            tr += e / float(sample.rsplit("uncorrected ", 1)[1].split()[0])
        est[wd] = es / tc
        raw[wd] = es / tr
    line = {"workload": workload, "partition": part, "rows": rows, "nnz": nnz,
            "full_pass_edges_per_s": full, "sampled_edges_per_s": est, "sampled_uncorrected_edges_per_s": raw,
            "sample_over_full": {wd: est[wd] / full[wd] for wd in widths},
            "uncorrected_over_full": {wd: raw[wd] / full[wd] for wd in widths},
            # one epoch's passes of the workload (edges x passes / summed time), as bench.py reports
            "epoch_sample_over_full": (sum(1 / full[wd] for wd in W.WORKLOADS[workload].passes() if wd in full) /
                                       sum(1 / est[wd] for wd in W.WORKLOADS[workload].passes() if wd in est)),
            "note": "1 core each; reference sgc_propagate (f64 column-major Eigen via oracle/_ref); the sampled "
                    "rate is what bench.py's cpu_baseline / --impl reference extrapolate from"}
    print(json.dumps(line), flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "ref_full_pass.json"), "w") as f:
        f.write(json.dumps(line) + "\n")


if __name__ == "__main__":
    main()
