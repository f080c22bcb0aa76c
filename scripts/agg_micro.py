"""K2 micro-benchmark on the bench workload's partition 0 (reddit_gcn, RMAT
scale 18, SPRING p=8): one SGC-normalised aggregation pass (self term, no
source scale) per width, kernel time from CUDA events on the launching stream,
algorithmic GB/s per SURVEY §8(d).  Env: WIDTHS=256,44,48 REPS=10."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_02300_b200 import gnnpart as gp
from benchdata import workloads as W  # noqa: E402

w = W.WORKLOADS[os.environ.get("WORKLOAD", "reddit_gcn")]
prep = W.prepare(w, lambda *a: None)
part = W.load_part(prep, int(os.environ.get("PART", 0)))
widths = [int(x) for x in os.environ.get("WIDTHS", "256,44,48").split(",")]
reps = int(os.environ.get("REPS", 10))
ctx = gp.Context(0)
out = {}
for width in widths:
    x = np.random.default_rng(0).standard_normal((part["ext"].size, width), dtype=np.float32)
    s = gp.Shard.from_part(part["ext"], part["owner"], part["role"], part["labels"], part["edges"], x, ctx)
    inf = s.info
    gp.sgc_propagate(s, 1)
    flush = os.environ.get("FLUSH") == "1"  # evict L2 before every pass (cold-input case)
    load = os.environ.get("TENSOR_LOAD") == "1"  # a tensor-core burst before every pass (power state)
    if flush or load:
        import torch
        junk = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        ma = torch.randn(8192, 8192, device="cuda", dtype=torch.bfloat16)
    ctx.set_kernel_timing(True)
    for _ in range(reps):
        if flush:
            torch.cuda.synchronize()
            junk.fill_(1)
            torch.cuda.synchronize()
        if load:
            for _ in range(int(os.environ.get("LOAD_N", "20"))):
                ma2 = ma @ ma
            torch.cuda.synchronize()
            if os.environ.get("LOAD_GAP_MS"):
                time.sleep(float(os.environ["LOAD_GAP_MS"]) / 1e3)
        gp.lib.catgnn_sgc_propagate(s.handle, 1)
    kt = ctx.kernel_time()
    ctx.set_kernel_timing(False)
    ms = kt["agg_ms"] / reps
    n, nnz = inf.rows, inf.nnz
    algo = nnz * (4 + 4 * width) + n * (4 * width * 2 + 8)
    out[width] = dict(us=round(ms * 1e3, 1), algo_gbs=round(algo / ms / 1e6), nnz=nnz, rows=n)
    s.close()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("CATGNN_")}, "k2": out}))
