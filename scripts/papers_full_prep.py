"""configs[3] at the full papers100M shape, host half (runs on any CPU host):
the RMAT stream (scale 27 = 134M ids, 1.6 B undirected records, the C++
generator, bit-identical to synth.rmat_edges_numpy) written as EDG1 and the
reference's own SPRING (upstream/_ref, unmodified) run over it for p = 16.
Saves the per-id home partition (u32) and SPRING's tau next to a manifest so
the GPU half (scripts/papers_full.py) regenerates the same stream and
completes / trains on the device.  ~25 min single-threaded SPRING.

    python scripts/papers_full_prep.py OUT_DIR
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SCALE = int(os.environ.get("PAPERS_SCALE", 27))
EDGES, SEED, BETA = 1_600_000_000, 4, 1.05
P = int(os.environ.get("PAPERS_P", 16))


def main():
    out = sys.argv[1]
    os.makedirs(out, exist_ok=True)
    from paper_2404_02300_b200 import synth
    from upstream.spring import spring_homes
    t0 = time.time()
    e, n, _ = synth.rmat_edges(SCALE, EDGES, seed=SEED)
    t1 = time.time()
    f = os.path.join(out, "edges.bin")
    with open(f, "wb") as fh:
        fh.write(b"EDG1")
        e.tofile(fh)
    del e
    t2 = time.time()
    home, tau = spring_homes(f, n, P, beta=BETA, tau_vol=0, seed=0)
    t3 = time.time()
    os.remove(f)
    np.save(os.path.join(out, "home.npy"), home)
    meta = dict(scale=SCALE, edges=EDGES, partitions=P, seed=SEED, beta=BETA, num_ids=int(n), tau_vol=int(tau),
                homed=int((home != 0xFFFFFFFF).sum()), part_homed=np.bincount(home[home != 0xFFFFFFFF],
                                                                               minlength=P).tolist(),
                times=dict(rmat=t1 - t0, write=t2 - t1, spring=t3 - t2))
    with open(os.path.join(out, "meta.json"), "w") as fh:
        json.dump(meta, fh)
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
