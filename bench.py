"""Benchmark of the per-partition GNN training step (BASELINE.json north star).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload reddit_gcn] [--sync S]
    (N > 1: launched under `python -m torch.distributed.run --nproc-per-node N ...
     bench.py --gpus N`, or started plainly with --gpus N, in which case bench.py
     re-executes itself under torch.distributed.run with N ranks; the world size
     must equal --gpus)

Workload (default, BASELINE.json configs[1]): 2-layer GCN (hidden 256) on the
reddit-shaped synthetic RMAT graph (scale 18, 57,307,946 undirected edges =
114.6M nnz, 602-d class-mean features, 41 classes) partitioned by the
reference's SPRING into p = 8 partitions with 1-hop completion.  Partitions
are assigned to ranks cyclically (8/N per GPU, strong scaling); one step = one
local iteration (full-batch forward + backward + Adam) over every partition of
the rank, followed by alpha-weighted model averaging (every --sync steps):
in-process across the rank's replicas and an NCCL all-reduce across ranks.

Metric: edges aggregated per second = sum over partitions and aggregation
passes of local nnz, per second of step time (max over ranks, CUDA events on
the library's stream).  Inputs stay resident in HBM for `value`; `e2e`
re-uploads the global feature matrix from pinned host memory through the C
ABI each step, gathers every partition's rows from it on the device (the
reference's gather-from-global load path, train.cpp:277-283) and reads the
loss back.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "edges aggregated/sec per epoch (local nnz x aggregation passes / step time)"
UNIT = "edges/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi style sampling of SM clocks and throttle reasons during the timed region."""

    def __init__(self, device=0, period=0.1):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self.device = period, device
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            names = {getattr(nv, k): k.replace("nvmlClocksEventReason", "").replace("nvmlClocksThrottleReason", "")
                     for k in dir(nv) if k.startswith(("nvmlClocksEventReason", "nvmlClocksThrottleReason"))
                     and isinstance(getattr(nv, k), int)}

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                        r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for bit, nm in names.items():
                            if bit and (r & bit) == bit and nm not in ("None", "All", "GpuIdle", "ApplicationsClocksSetting"):
                                self.reasons.add(nm)
                    except Exception:
                        pass
                    time.sleep(self.period)
            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception as e:  # pragma: no cover
            log("[clocks] unavailable:", e)
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def self_launch(gpus):
    """`python bench.py --gpus N` without a launcher: re-execute this command as N
    ranks under torch.distributed.run (one process per GPU, 127.0.0.1
    rendezvous) and return its exit code.  NCCL_DEBUG=INFO (INIT subsystem) so
    the communicator's rank count is visible in the log."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(gpus),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__)]
    cmd += sys.argv[1:]
    log(f"[bench] --gpus {gpus} without a launcher: {' '.join(cmd)}")
    return subprocess.call(cmd, env=env)


def act_width(d):
    """Row stride of a device activation (gnn.cu act_width): 16-float multiples below 128."""
    return (d + 15) // 16 * 16 if d < 128 else (d + 3) // 4 * 4


def agg_bytes(nnz, rows, width, self_term, eb=4):
    """nnz*(4 + 4d) + N*(4d*(1+self) + 8), with the gathered
    input rows at eb bytes per element (2: fp16 passes): nnz*(4 + eb*d) +
    N*(eb*d*self + 4d + 8)."""
    return nnz * (4 + eb * width) + rows * (eb * width * self_term + 4 * width + 8)


def load_ncu_traffic(w):
    """ncu DRAM / L2 bytes of every K2 launch of one step of this workload
    (profiles/r02_k2_traffic_<workload>.json, scripts/k2_traffic.py: an ncu
    metric pass over the same bench command), or None."""
    p = os.path.join(ROOT, "profiles", f"r02_k2_traffic_{w.name}.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        if d.get("workload_key") == w.key():
            return d
    return None


def k2_roofline(w, mine, part_nnz, part_rows, agg_ms_step, agg_launches, ms_step, hbm, hbm_src, l2_gbs, hbm_rd,
                views=None):
    """Roofline of K2 whose every number is a fraction of the peak it is divided by:
    * effective_gbs: SURVEY §8(d) algorithmic bytes (nnz*(4+4d) + N*(4d(1+self)+8)
      per pass) / in-step K2 time.  Each gathered row counts once per edge, so on
      RMAT hubs this exceeds what DRAM moves: it is what the SMs pull through L2.
    * dram_gbs: ncu DRAM bytes of the same launches / the same in-step time.
    * bound "hbm" when the DRAM rate is near the HBM peak (dram_frac >= 0.75),
      else "l2" when the effective rate exceeds the HBM peak (the gathers are
      served from L2: the ceiling is the measured L2 read rate), else "hbm"."""
    self_term = {"gcn": 1, "gin": 1, "sage": 0}[w.model]
    widths = list(zip(w.passes(), w.pass_elem_bytes(), w.lean_pass_views()))

    def gathered(k, kind):  # (nnz, rows) a pass of partition k gathers (lean train-step views)
        nz, rw = part_nnz[k], part_rows[k]
        if views is not None and kind == "train_rows":
            return views[k][1], views[k][0]
        if views is not None and kind == "train_nbrs":
            return views[k][2], rw
        return nz, rw
    algo = sum(agg_bytes(*gathered(k, kind), wd, self_term, eb)
               for k in range(len(part_nnz)) for wd, eb, kind in widths)
    # compulsory: every input row of the shard once, indices and offsets once, each output row once
    comp = sum(eb * wd * part_rows[k] + 4 * wd * gathered(k, kind)[1] + 4 * gathered(k, kind)[0]
               + 8 * (gathered(k, kind)[1] + 1) for k in range(len(part_nnz)) for wd, eb, kind in widths)
    t = agg_ms_step / 1e3
    eff = algo / t / 1e9 if t > 0 else None
    ncu = load_ncu_traffic(w)
    dram = l2b = None
    if ncu:
        mine_set = set(mine)
        recs = [r for r in ncu["launches"] if r["partition"] in mine_set]
        dram = sum(r["dram_bytes"] for r in recs)
        l2b = sum(r["l2_bytes"] for r in recs)
    dram_gbs = dram / t / 1e9 if (dram and t > 0) else None
    dram_frac = dram_gbs / hbm if dram_gbs else None
    if dram_frac is not None and dram_frac >= 0.75:
        bound = "hbm"
    elif eff and eff > hbm and l2_gbs:
        bound = "l2"
    else:
        bound = "hbm"
    if bound == "l2":
        achieved, peak, src = eff, l2_gbs, ("catgnn_probe_read_bandwidth: 64 MB buffer, 128-bit ld.global.cg, "
                                            "50 passes, best of 3 (measured L2 read rate, same device)")
    else:
        achieved, peak, src = (dram_gbs if dram_gbs else eff), hbm, f"MEASURED_PEAKS.json hbm_gbs ({hbm_src})"
    per_launch = max(agg_launches, 1)
    return {"bound": bound, "kernel": "catgnn::agg_kernel (K2 neighbourhood aggregation)",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak if achieved else None,
            "traffic": dram / per_launch if dram else None, "peak_source": src,
            "effective_gbs": eff, "algorithmic_bytes_per_step": algo,
            "algorithmic_bytes_per_launch": algo / per_launch,
            "dram_bytes_per_step": dram, "dram_gbs": dram_gbs, "dram_frac": dram_frac,
            "hbm_peak_gbs": hbm, "hbm_read_probe_gbs": hbm_rd,
            "l2_read_peak_gbs": l2_gbs, "l2_frac": eff / l2_gbs if (eff and l2_gbs) else None,
            "l2_bytes_per_step_ncu": l2b,
            "compulsory_bytes_per_step": comp, "dram_over_compulsory": dram / comp if dram else None,
            "launches_per_step": agg_launches, "agg_ms_per_step": agg_ms_step,
            "agg_share_of_step": agg_ms_step / ms_step,
            "traffic_source": (ncu["source"] if ncu else "no ncu capture for this workload "
                               "(profiles/r02_k2_traffic_<workload>.json)"),
            "note": "frac = achieved / peak of the bound that applies; effective_gbs counts every gathered "
                    "row per edge (SURVEY §8(d) bytes) and exceeds the DRAM peak when rows are re-served "
                    "from L2; dram_* are ncu DRAM bytes over the in-step K2 time"}


def reference_jobs(prep, samples, budget_edges):
    """Bounded samples for the reference CPU path: samples = [(partition,
    block)].  Each sample is a SELF-CONTAINED row-block subgraph: the rows
    [R0, R1) holding the block-th ~budget_edges local edges of the partition
    CSR (the reference's own build_adjacency) keep their neighbour lists, and
    the rows they gather from are renumbered after them with empty lists — so
    the reference's per-row loop runs over the sample's rows plus its gather
    sources only, not over the whole partition (whose other rows' edges the
    sample does not count)."""
    from oracle import ref
    jobs, csr = [], {}
    for i, blk in samples:
        if i not in csr:
            d = prep["dir"]
            edges = np.load(os.path.join(d, f"p{i}_edges.npy"))
            ext = np.load(os.path.join(d, f"p{i}_ext.npy"))
            local = np.searchsorted(ext, edges.ravel()).astype(np.uint32).reshape(-1, 2)
            csr[i] = (ext.size,) + tuple(ref.build_adjacency(ext.size, local))
        rows, off, nb = csr[i]
        # block indices past a small partition's edges wrap around (every
        # sample is a non-empty row range of the partition)
        blk %= max(1, -(-int(off[rows]) // budget_edges))
        R0 = min(int(np.searchsorted(off, blk * budget_edges)), max(rows - 1, 0))
        R1 = max(R0 + 1, min(int(np.searchsorted(off, (blk + 1) * budget_edges)), rows))
        nbs = nb[off[R0]: off[R1]].astype(np.int64)
        ns = R1 - R0
        # compact ids: sampled rows 0..ns-1, then the other gather sources
        others = np.setdiff1d(np.unique(nbs), np.arange(R0, R1))
        remap = np.where((nbs >= R0) & (nbs < R1), nbs - R0, ns + np.searchsorted(others, nbs))
        rows_c = ns + others.size
        off_c = np.empty(rows_c + 1, np.uint32)
        off_c[:ns + 1] = (off[R0:R1 + 1] - off[R0]).astype(np.uint32)
        off_c[ns + 1:] = off_c[ns]
        jobs.append((rows_c, off_c, remap.astype(np.uint32), int(off[R1] - off[R0]), ns))
    return jobs


def cpu_reference_rate(w, jobs, seed=0):
    """The reference's aggregation (proj/src/train.cpp:49-65 sgc_propagate, compiled
    unmodified via oracle/_ref) over the bounded samples, one pass per width of
    this workload's epoch schedule; one host thread per partition sample (the
    reference is single-threaded and its workers are schedule-independent).

    A sample's gather-source rows cost the reference its per-row work (copy
    and scale of a strided row) without contributing edges, which a full pass
    amortises over every row's own neighbours; that share is measured on the
    same sample with no edges (rows only) and removed: time = t(sample) -
    t(rows only) * U / rows, U = gather-source rows.  scripts/ref_full_pass.py
    checks the estimate against a whole-partition pass."""
    from oracle import ref
    widths = w.passes()
    results = [None] * len(jobs)

    def run(j):
        rows, off_s, nb_s, edges_s, ns = jobs[j]
        rng = np.random.default_rng(seed + j)
        t = t_raw = 0.0
        empty = np.zeros_like(off_s)
        for wd in widths:
            x = rng.standard_normal(rows * wd)  # column-major f64 (Eigen MatrixXd)
            t0 = time.perf_counter()
            ref.sgc_propagate_colmajor(off_s, nb_s, x, rows, wd, 1)
            ts = time.perf_counter() - t0
            t0 = time.perf_counter()
            ref.sgc_propagate_colmajor(empty, nb_s[:1], x, rows, wd, 1)
            t_rows = time.perf_counter() - t0
            t_raw += ts
            t += max(ts - t_rows * (rows - ns) / rows, 0.25 * ts)
        results[j] = (edges_s * len(widths), t, t_raw)

    ths = [threading.Thread(target=run, args=(j,)) for j in range(len(jobs))]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    edges = sum(r[0] for r in results)
    wall = max(r[1] for r in results)
    raw = edges / max(r[2] for r in results)
    sample = (f"reference sgc_propagate (1 hop) over {len(jobs)} self-contained row-block subgraph(s) of "
              f"~{jobs[0][3]} local edges ({jobs[0][4]} rows + {jobs[0][0] - jobs[0][4]} gather-source rows "
              f"in the first), distinct row blocks of the partitions round-robin, one pass per epoch width "
              f"{widths}, f64 column-major (Eigen MatrixXd), {len(jobs)} host thread(s), one block each; "
              f"gather-source rows' per-row time (measured rows-only) removed: uncorrected {raw:.4g} edges/s")
    return edges / wall, len(jobs), sample


def run_reference(args, w, prep):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    # every host thread: the reference is single-threaded and its workers are
    # schedule-independent, so blocks of the partitions run side by side
    threads = os.cpu_count() or 1
    jobs = reference_jobs(prep, [(t % w.partitions, t // w.partitions) for t in range(threads)], args.ref_edges)
    vals = []
    for s in range(args.warmup + args.steps):
        v, cores, sample = cpu_reference_rate(w, jobs, seed=s)
        if s >= args.warmup:
            vals.append(v)
    value = float(np.median(vals))
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(w, prep, args), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def gemm_precision(w):
    """K3 operand precision per layer kind (gnn.cu bf_layer): transform-first
    GCN / GIN layers run bf16x3 kind::f16 MMAs, the others 3xTF32 kind::tf32."""
    kinds = []
    for l in range(w.layers):
        d_in = w.dim if l == 0 else w.hidden
        d_out = w.classes if l + 1 == w.layers else w.hidden
        agg_first = d_in <= d_out if w.model == "sage" else d_in < d_out
        kinds.append("bf16x3 (tcgen05 kind::f16)" if w.model != "sage" and not agg_first
                     else "3xTF32 (tcgen05 kind::tf32)")
    return kinds


def dtype_label(w):
    eb = w.pass_elem_bytes()
    agg = ("fp32 accumulation; gathered inputs " +
           ("fp32" if all(e == 4 for e in eb) else
            "fp16 on the passes " + ", ".join(str(x) for x, e in zip(w.passes(), eb) if e == 2) +
            " (guarded forward / scaled gradients), fp32 otherwise"))
    return f"f32 ({'/'.join(sorted(set(gemm_precision(w))))} tensor-core GEMMs; aggregation: {agg})"


def workload_config(w, prep, args):
    m = prep["meta"]
    return {"workload": w.name, "gnn": f"{w.layers}-layer {w.model.upper()} hidden {w.hidden}",
            "graph": f"RMAT scale {w.scale}, {w.edges} undirected edges ({m['nnz']} nnz), |V|={m['num_nodes']}",
            "feature_dim": w.dim, "classes": w.classes, "partitions": w.partitions,
            "partitioner": f"reference SPRING beta={w.beta} tau_vol={m['tau_vol']} + 1-hop completion",
            "replication_factor": m["rf"], "part_nnz": m["part_nnz"], "sum_over_max_edges": m["sum_over_max"],
            "aggregation_widths": w.passes(),
            "aggregation_row_stride_floats": [act_width(x) for x in w.passes()],
            "aggregation_input_bytes_per_element": w.pass_elem_bytes(), "sync_interval": args.sync,
            "optimizer": "adam lr 0.01", "gemm_precision": gemm_precision(w),
            "step": "one full-batch local iteration per partition + averaging",
            "partitions_per_gpu": w.partitions // max(1, dist_env()[0]),
            "l2": "inputs larger than L2 (per-partition features 0.5 GB, activations > 126 MB)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=os.environ.get("CATGNN_WORKLOAD", "reddit_gcn"))
    ap.add_argument("--sync", type=int, default=1)
    ap.add_argument("--ref-edges", type=int, default=300_000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--lanes", type=int, default=int(os.environ.get("CATGNN_LANES", "2")),
                    help="shard lanes: partitions of a rank trained on this many concurrent streams")
    ap.add_argument("--agg-sms", type=int, default=int(os.environ.get("CATGNN_LANE_AGG_SMS", "0")),
                    help="with lanes > 1: SMs a K2 grid covers (0 = all)")
    ap.add_argument("--gemm-sms", type=int, default=int(os.environ.get("CATGNN_LANE_GEMM_SMS", "0")),
                    help="with lanes > 1: SMs a K3 grid uses (0 = all)")
    ap.add_argument("--graph", type=int, default=int(os.environ.get("CATGNN_GRAPH", "1")),
                    help="replay the device-resident step as one CUDA graph (1) or enqueue it eagerly (0)")
    args = ap.parse_args()

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        raise SystemExit(self_launch(args.gpus))
    from benchdata import workloads as W
    w = W.WORKLOADS[args.workload]
    world, rank, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"world size {world} (WORLD_SIZE) != --gpus {args.gpus}: launch one rank per GPU")
    if args.impl == "reference":
        if rank == 0:
            # NumPy RMAT: the reference arm's process never loads libcatgnn.so
            prep = W.prepare(w, log, native=False)
            run_reference(args, w, prep)
        return

    import torch
    import torch.distributed as dist
    # CATGNN_BENCH_HOST_COLLECTIVES=1: validation mode for the multi-rank flow on a
    # single-GPU box (ranks share the device, gloo on the host replaces NCCL)
    host_coll = os.environ.get("CATGNN_BENCH_HOST_COLLECTIVES") == "1"
    ndev = torch.cuda.device_count()
    if world > ndev and not host_coll:
        # more ranks than GPUs (e.g. --gpus 2 on a one-GPU box): NCCL refuses two
        # ranks on one device, so the ranks share the GPUs and collectives go through
        # gloo on the host; the line says so (config.shared_devices)
        log(f"[bench] {world} ranks on {ndev} GPU(s): ranks share devices, host (gloo) collectives")
        host_coll = True
    if host_coll:
        local = local % max(1, ndev)
    torch.cuda.set_device(local)
    if world > 1:
        if host_coll:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    if w.partitions % world:
        raise SystemExit(f"partition count {w.partitions} must be a multiple of the GPU count {world}")
    # data preparation (untimed; rank 0 builds the cache, the others wait)
    if rank == 0:
        prep = W.prepare(w, log)
    if world > 1:
        dist.barrier()
    if rank != 0:
        prep = W.prepare(w, log)
    meta = prep["meta"]

    from paper_2404_02300_b200 import gnnpart as gp
    from paper_2404_02300_b200.gnn import ADAM, Comm, GNNModel, model_average, sync_weights, weighted_sum
    stream = torch.cuda.Stream()
    ctx = gp.Context(local, stream.cuda_stream)
    # shard lanes: partition k of this rank trains on lane k % L (own stream and
    # scratch), so one partition's aggregation overlaps another's GEMMs
    lanes = max(1, min(args.lanes, w.partitions // world))
    lane_streams = [stream] + [torch.cuda.Stream() for _ in range(lanes - 1)]
    ctxs = [ctx] + [gp.Context(local, st.cuda_stream) for st in lane_streams[1:]]
    if lanes > 1:
        for c in ctxs:
            c.set_sm_budget(args.agg_sms, args.gemm_sms)
    mine = list(range(rank, w.partitions, world))
    X = np.load(os.path.join(prep["dir"], "features.npy"), mmap_mode="r")
    labels = np.load(os.path.join(prep["dir"], "labels.npy"))
    shards = []
    t0 = time.time()
    for k, i in enumerate(mine):
        p = W.load_part(prep, i, X, labels)
        s = gp.Shard.from_part(p["ext"], p["owner"], p["role"], p["labels"], p["edges"], p["features"],
                               ctxs[k % lanes])
        shards.append(s)
    # e2e input: the global feature matrix in pinned host memory, refreshed into
    # the device feature store every step; shards gather their rows from it
    host_X = torch.empty(X.shape, dtype=torch.float32, pin_memory=True)
    host_X.numpy()[:] = X
    # two device stores on a copy stream: step t+1's upload overlaps step t's
    # work (the library orders uploads and gathers with events)
    copy_ctx = gp.Context(local) if not args.no_e2e else None
    # N > 1 (NCCL): each rank uploads 1/N of the rows over its own host link and an
    # in-place NCCL all-gather over NVLink completes every rank's store
    shard_feats = world > 1 and not host_coll and not args.no_e2e
    rows_per_rank = -(-X.shape[0] // world)
    store_rows = rows_per_rank * world if shard_feats else X.shape[0]
    stores = [gp.FeatureStore(store_rows, X.shape[1], copy_ctx) for _ in range(2)] if not args.no_e2e else None
    log(f"[rank {rank}] {len(shards)} shards resident in {time.time() - t0:.1f}s")
    counts_all = meta["part_train"]
    alpha_all = sync_weights(counts_all)
    my_alpha = [alpha_all[i] for i in mine]
    my_counts = [counts_all[i] for i in mine]
    shared_devices = world > ndev
    comm = None
    feat_comm = None
    if world > 1 and not host_coll:
        uid = [Comm.unique_id() if rank == 0 else None, Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = Comm(ctx, world, rank, uid[0])
        if shard_feats:  # its own communicator on the copy stream
            feat_comm = Comm(copy_ctx, world, rank, uid[1])

    def refresh_features(store):
        """This step's input features from pinned host memory into a device store."""
        if feat_comm is None:
            store.upload(host_X.numpy())
        else:
            lo = rank * rows_per_rank
            hi = min(X.shape[0], lo + rows_per_rank)
            if hi > lo:
                store.upload(host_X.numpy()[lo:hi], row_begin=lo)
            store.allgather(feat_comm, rows_per_rank)
    kw = dict(optimizer=ADAM, lr=0.01, seed=0, ctx=ctx)
    shared = GNNModel(w.model, w.layers, w.dim, w.hidden, w.classes, **kw)
    reps = [GNNModel(w.model, w.layers, w.dim, w.hidden, w.classes, **dict(kw, ctx=ctxs[k % lanes]))
            for k in range(len(shards))]
    for r in reps:
        r.copy_params_from(shared)

    def average():
        if world == 1:
            model_average(reps, my_counts, shared)
        else:
            # this rank's share sum_i alpha_i theta_i with the GLOBAL alphas (a
            # rank without train rows contributes zeros), then the all-reduce
            weighted_sum(reps, my_alpha, shared)
            if comm is not None:
                shared.allreduce(comm)  # C1: NCCL all-reduce on the library stream
            else:  # host-collective validation mode
                t = torch.from_numpy(shared.get_params())
                dist.all_reduce(t)
                shared.set_params(t.numpy())
        for r in reps:
            r.copy_params_from(shared)

    state = {"it": 0}

    def step(e2e=False, t=0, n=1, serial=False):
        losses = []
        for c in ctxs[1:]:  # fork the lanes off the main stream (graph capture needs it)
            c.wait_for(ctx)
        prev = ctx
        if e2e:
            if t == 0:
                refresh_features(stores[0])
            if t + 1 < n:  # prefetch the next step's inputs on the copy stream
                refresh_features(stores[(t + 1) % 2])
        for k, (r, s) in enumerate(zip(reps, shards)):
            if serial:  # lanes in turn: per-kernel event times without overlap
                ctxs[k % lanes].wait_for(prev)
                prev = ctxs[k % lanes]
            if e2e:
                s.gather_features(stores[t % 2])
            r.train_step(s, want_loss=False)
        if e2e:  # the step's result back on the host: one sync after every replica's step
            losses = [r.last_loss() for r in reps]
        state["it"] += 1
        if state["it"] % args.sync == 0:
            average()
        for c in ctxs[1:]:  # join the lanes back into the main stream
            ctx.wait_for(c)
        return losses

    def timed(n, e2e=False, graph=None):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        wall0 = time.perf_counter()
        if graph is not None:
            with torch.cuda.stream(stream):
                for t in range(n // args.sync):
                    graph.replay()
        else:
            for t in range(n):
                step(e2e, t, n)
        ev1.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - wall0
        ms = ev0.elapsed_time(ev1)
        if e2e:
            ms = max(ms, wall * 1e3)  # host-side copies/syncs are part of the end-to-end time
        if world > 1:
            t = torch.tensor([ms], device="cpu" if host_coll else "cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # CUDA graph of one averaging period (s local iterations + the average):
    # the step's ~180 launches replayed without host work between them
    # (not in the host-collective validation mode: its gloo all-reduce syncs the host)
    use_graph = bool(args.graph) and args.steps % args.sync == 0 and not host_coll
    def timing(on):
        for c in ctxs:
            c.set_kernel_timing(on)

    def launch_count():
        return sum(c.launches for c in ctxs)

    timing(True)  # warm the event pool before a capture
    def timed_e2e_graph(n, diag=False):
        """End-to-end steps as replays of one CUDA graph holding two steps: step
        2i gathers from store 0 while store 1 receives step 2i+1's features on
        the copy stream, step 2i+1 gathers from store 1 while store 0 receives
        the next replay's; every step's losses are copied into pinned host
        memory and read after the replay.  The first step's upload runs eagerly
        inside the timed region."""
        R = len(reps)
        host_loss = torch.zeros(2 * R, dtype=torch.float64).pin_memory()
        base = host_loss.data_ptr()
        rows = [0] * (2 * R)
        torch.cuda.synchronize()
        for st in stores:
            st.reset_deps()
        if diag:
            timing(True)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream, capture_error_mode="thread_local"):
            copy_ctx.wait_for(ctx)
            for c in ctxs[1:]:
                c.wait_for(ctx)
            for sub in (0, 1):
                refresh_features(stores[1 - sub])  # the next step's inputs (copy stream)
                for k, (r, s) in enumerate(zip(reps, shards)):
                    s.gather_features(stores[sub])
                    r.train_step(s, want_loss=False)
                    rows[sub * R + k] = r.last_loss_async(base + 8 * (sub * R + k))
                average()
            ctx.wait_for(copy_ctx)
            for c in ctxs[1:]:
                ctx.wait_for(c)
        for st in stores:
            st.reset_deps()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        wall0 = time.perf_counter()
        refresh_features(stores[0])  # step 0's inputs
        ctx.wait_for(copy_ctx)
        losses = []
        with torch.cuda.stream(stream):
            for _ in range(n // 2):
                g.replay()
                stream.synchronize()  # both steps' losses are on the host now
                hl = host_loss.tolist()
                losses.append([hl[j] / rows[j] if rows[j] else 0.0 for j in range(2 * R)])
        ev1.record(stream)
        torch.cuda.synchronize()
        ms = max(ev0.elapsed_time(ev1), (time.perf_counter() - wall0) * 1e3)
        if world > 1:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        if not all(np.isfinite(x).all() for x in losses):
            raise RuntimeError("non-finite loss in the e2e steps")
        return ms

    for _ in range(args.warmup):
        step()
    # finish the averaging period, so every lazily sized buffer (the averaging
    # scratch included) exists before a graph capture
    while state["it"] % args.sync:
        step()
    torch.cuda.synchronize()
    timing(True)
    graph = None
    launches0 = launch_count()
    if use_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream, capture_error_mode="thread_local"):
                for _ in range(args.sync):
                    step()
            launches_per_replay = launch_count() - launches0
        except Exception as ex:  # pragma: no cover - fall back to eager launches
            log(f"[rank {rank}] CUDA graph capture failed ({ex}); timing eager steps")
            graph = None
            torch.cuda.synchronize()
            timing(True)
            launches0 = launch_count()
    with ClockSampler(local) as clk:
        total_ms = timed(args.steps, graph=graph)
    launches_eager = launch_count() - launches0
    if lanes > 1:
        # concurrent lanes overlap kernels, so their event times would add up
        # to more than the step: the per-kernel breakdown and the roofline come
        # from one averaging period run with the lanes in turn (eager)
        timing(False)
        timing(True)
        for _ in range(args.sync):
            step(serial=True)
        torch.cuda.synchronize()
        graph_for_records = None
    else:
        graph_for_records = graph
    # per-kernel CUDA events: every launch of the timed region (eager), or the
    # graph's event nodes as recorded by its last replay (one averaging period)
    # (with lanes > 1 kernels of different lanes overlap: their event times add up
    # to more than the step and each includes the time it shared the GPU)
    kts = [c.kernel_time() for c in ctxs]
    kt = {k: sum(x[k] for x in kts) for k in kts[0]}
    timed_steps = args.sync if (graph_for_records is not None or lanes > 1) else args.steps
    recs = {}
    for c in ctxs:
        for k, v in c.kernel_records().items():
            a = recs.get(k, (0.0, 0))
            recs[k] = (a[0] + v[0], a[1] + v[1])
    breakdown = {k: {"ms_per_step": round(v[0] / timed_steps, 4), "launches_per_step": v[1] / timed_steps}
                 for k, v in sorted(recs.items(), key=lambda kv: -kv[1][0])}
    timing(False)
    launches = launches_per_replay * (args.steps // args.sync) if graph is not None else launches_eager
    ms_step = total_ms / args.steps

    widths = w.passes()  # logical widths: algorithmic bytes exclude the row padding
    part_nnz = [meta["part_nnz"][i] for i in mine]
    part_rows = [meta["part_rows"][i] for i in mine]
    edges_per_step_rank = sum(part_nnz) * len(widths)
    edges_per_step = sum(meta["part_nnz"]) * len(widths)
    value = edges_per_step * args.steps / (total_ms / 1e3)

    # roofline of the dominant kernel (K2) from per-launch CUDA events
    agg_ms_step = kt["agg_ms"] / timed_steps
    hbm, bf16, src = peaks()
    per_launch = kt["agg_launches"] / timed_steps
    # L2 / HBM read-rate probes (same device, after the timed region)
    l2_gbs = hbm_rd_gbs = None
    try:
        l2_gbs = max(gp.probe_read_bandwidth(64 << 20, 50, ctx) for _ in range(3))
        hbm_rd_gbs = max(gp.probe_read_bandwidth(4 << 30, 3, ctx) for _ in range(2))
    except Exception as ex:  # pragma: no cover
        log("[probe] failed:", ex)
    views = [s.train_views() for s in shards]  # (train rows, their nnz, nnz into train rows) per partition
    if os.environ.get("CATGNN_VIEWS_OUT"):  # scripts/k2_traffic.py: per-pass gathered rows / nnz
        with open(os.environ["CATGNN_VIEWS_OUT"], "w") as f:
            json.dump(views, f)
    roofline = k2_roofline(w, mine, part_nnz, part_rows, agg_ms_step, per_launch, ms_step, hbm, src, l2_gbs,
                           hbm_rd_gbs, views)
    gathered_per_step = sum(
        (v[1] if kind == "train_rows" else v[2] if kind == "train_nbrs" else nz)
        for nz, v in zip(part_nnz, views) for kind in w.lean_pass_views())
    # useful GEMM flops per step: forward + weight gradient (+ input gradient past layer 0)
    gemm_flops = 0
    for rows_i in part_rows:
        d_in = w.dim
        for l in range(w.layers):
            d_out = w.classes if l + 1 == w.layers else w.hidden
            k = 2 * d_in if w.model == "sage" else d_in
            gemm_flops += 2 * rows_i * k * d_out * (3 if l > 0 else 2)
            d_in = d_out
    gemm = {"kernel": "catgnn::gemm_tf32_kernel (K3 tcgen05; " + ", ".join(sorted(set(gemm_precision(w)))) + ")",
            "ms_per_step": kt["gemm_ms"] / timed_steps,
            "achieved_tflops": gemm_flops / (kt["gemm_ms"] / timed_steps / 1e3) / 1e12 if kt["gemm_ms"] else None,
            "achieved_is": "useful flops (2MNK); the split-precision schemes issue 3 MMAs per product",
            "peak_tflops_bf16": bf16, "peak_note": "measured dense bf16 (MEASURED_PEAKS.json); kind::tf32 runs at half"}

    # end-to-end through the C ABI: global features re-uploaded from pinned host memory each step, loss read back
    e2e = None
    # the first layer's GEMMs read the bf16x3 feature copy: gathers write only that
    split_only = w.model in ("gcn", "gin") and w.dim > w.hidden and os.environ.get("CATGNN_GEMM_BF16X3", "1") != "0"
    if not args.no_e2e and split_only:
        for s in shards:
            s.set_feature_layout(True)
    if not args.no_e2e:
        for t in range(2):
            step(True, t, 2)
        diag = os.environ.get("CATGNN_E2E_BREAKDOWN") == "1"  # per-kernel times of the e2e steps
        e2e_graph = use_graph and graph is not None and args.sync == 1 and args.steps % 2 == 0
        if e2e_graph:
            try:
                e2e_ms = timed_e2e_graph(args.steps, diag) / args.steps
            except Exception as ex:  # pragma: no cover - fall back to eager steps
                log(f"[rank {rank}] e2e graph failed ({ex}); timing eager e2e steps")
                torch.cuda.synchronize()
                for st in stores:
                    st.reset_deps()
                e2e_graph = False
        if not e2e_graph:
            if diag:
                timing(True)
            e2e_ms = timed(args.steps, e2e=True) / args.steps
        if diag:
            for c in ctxs:
                for k, v in sorted(c.kernel_records().items(), key=lambda kv: -kv[1][0]):
                    log(f"[e2e] {k}: {v[0] / (2 if e2e_graph else args.steps):.3f} ms/step, "
                        f"{v[1] / (2 if e2e_graph else args.steps):.1f} launches/step")
            timing(False)
        h2d = int(host_X.numel()) * 4 * (1 if feat_comm is not None else world)
        e2e = {"value": edges_per_step / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": 8 * w.partitions, "ms_per_step": e2e_ms,
               "graph": "two steps per CUDA graph replay (device stores alternate)" if e2e_graph else None,
               "feature_layout": "bf16x3 (hi, lo) rows written by the gather" if split_only else "fp32 rows",
               "path": "catgnn_features_upload (global features, pinned H2D on a copy stream, double-buffered; "
                       "N > 1: 1/N of the rows per rank + catgnn_features_allgather over NVLink; "
                       "step t+1's copy overlaps step t) + per partition catgnn_shard_gather_features + "
                       "catgnn_model_train_step; every partition's loss D2H every step "
                       "(catgnn_model_last_loss_async into pinned memory, read on the host after each replay); "
                       "model averaging"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample = cpu_reference_rate(w, reference_jobs(prep, [(0, 0)], args.ref_edges))
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample}

    if rank == 0:
        cfg = workload_config(w, prep, args)
        if host_coll:
            cfg["collectives"] = "host (gloo): validation mode, not an NVLink measurement"
            cfg["shared_devices"] = bool(shared_devices)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": dtype_label(w),
                "data": "synthetic (RMAT + reference SPRING partitions, random-init weights)",
                "config": cfg, "roofline": roofline, "gemm": gemm,
                "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "step_breakdown": breakdown,
                "lanes": lanes, "kernel_times_from": ("one averaging period with the lanes in turn (per-kernel CUDA "
                                                      "events without lane overlap)" if lanes > 1 else
                                                      "the timed region's CUDA events"),
                "global_nnz_edges_per_s": meta["nnz"] * len(widths) * args.steps / (total_ms / 1e3),
                "value_definition": ("local nnz x aggregation passes per step / step time: the epoch's "
                                     "full-graph-equivalent aggregation; a train step gathers the last "
                                     "layer's passes only over its train-row views (same results)"),
                "edges_gathered_per_step_rank": gathered_per_step,
                "edges_equivalent_per_step_rank": edges_per_step_rank,
                "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    if feat_comm is not None:
        feat_comm.close()
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
