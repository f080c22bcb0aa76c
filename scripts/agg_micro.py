"""K2 micro-benchmark: one SGC aggregation pass over an RMAT shard, kernel time
from CUDA events on the launching stream, algorithmic GB/s."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_02300_b200 import gnnpart as gp, synth  # noqa: E402

scale = int(os.environ.get("SCALE", 18))
edges = int(os.environ.get("EDGES", 14_000_000))
t0 = time.time()
e, n, _ = synth.rmat_edges(scale, edges, seed=42)
print(f"gen {time.time()-t0:.1f}s rows={n} edges={edges}", flush=True)
ctx = gp.Context(0)
out = {}
for width in [256, 48, 64, 604]:
    x = np.random.default_rng(0).standard_normal((n, width), dtype=np.float32)
    t0 = time.time()
    s = gp.Shard.from_edges(n, e.astype(np.uint32), x, ctx)
    inf = s.info
    build_s = time.time() - t0
    gp.sgc_propagate(s, 1)
    ctx.set_kernel_timing(True)
    reps = 5
    for _ in range(reps):
        gp.lib.catgnn_sgc_propagate(s.handle, 1)
    kt = ctx.kernel_time()
    ms = kt["agg_ms"] / reps
    nnz = inf.nnz
    ld = (width + 3) // 4 * 4
    algo = nnz * (4 + 4 * ld) + n * (4 * ld * 2 + 8)
    out[width] = dict(ms=ms, gbs=algo / ms / 1e6, nnz=nnz, heavy=inf.heavy_rows, units=inf.tasks, build_s=build_s)
    print(width, out[width], flush=True)
    ctx.set_kernel_timing(False)
    s.close()
print(json.dumps(out))
