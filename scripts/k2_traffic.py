"""DRAM / L2 traffic of every K2 aggregation launch of one bench step (ncu
metric pass, not --set full), summarised per pass and per step for the bench
line's roofline (all passes, not 2 of 32).

    python scripts/k2_traffic.py [WORKLOAD] [OUT.json]

Runs `ncu --metrics ... -k regex:agg_ python bench.py --steps 1 --warmup 1
--graph 0 --no-e2e --no-cpu-baseline --lanes 1` (one eager warm-up step + one timed
step, partitions in order on one stream),
keeps the timed step's launches (the second half), and tags each agg_kernel
launch with its partition and pass (the step runs partitions in order, each
with its epoch's passes in workload.passes() order; split-row fix-ups are
folded into the pass they finish).  ncu replays every kernel with caches
flushed, so its times are cold and serialised: the bench line uses the DRAM
bytes from here and its own in-step CUDA-event times.
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
           "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-3, "usecond": 1,
         "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6, "%": 1, "": 1}


def compulsory_bytes(nnz, rows_in, rows, width, eb):
    """Each input row read once (eb bytes per element; all rows_in of the shard,
    an upper bound for a train-row view), column indices and row offsets once,
    each output row written once (what an infinite cache would move)."""
    return eb * width * rows_in + 4 * width * rows + 4 * nnz + 8 * (rows + 1)


def main():
    workload = sys.argv[1] if len(sys.argv) > 1 else "reddit_gcn"
    out = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", f"r02_k2_traffic_{workload}.json")
    from benchdata import workloads as W
    w = W.WORKLOADS[workload]
    prep = W.prepare(w, lambda *a: None)
    meta = prep["meta"]
    log = os.environ.get("K2_TRAFFIC_CSV") or os.path.join(ROOT, "gpurun_out", f"k2_traffic_{workload}.csv")
    if not os.environ.get("K2_TRAFFIC_CSV"):  # else: re-summarise an existing capture
        os.makedirs(os.path.dirname(log), exist_ok=True)
        env = dict(os.environ, CATGNN_WORKLOAD=workload, CATGNN_VIEWS_OUT=log + ".views.json")
        cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "-k", "regex:agg_", "--csv",
               "--log-file", log, sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "1",
               "--graph", "0", "--no-e2e", "--no-cpu-baseline", "--lanes", "1"]
        subprocess.run(cmd, env=env, check=True, stdout=subprocess.DEVNULL)
    launches = {}
    with open(log) as f:
        text = f.read()
    text = text[text.index('"ID"'):]
    for r in csv.DictReader(io.StringIO(text)):
        k = int(r["ID"])
        d = launches.setdefault(k, {"kernel": r["Kernel Name"]})
        v = float(r["Metric Value"].replace(",", "")) * SCALE.get(r["Metric Unit"], 1)
        d[r["Metric Name"]] = v
    seq = [launches[k] for k in sorted(launches)]
    seq = seq[len(seq) // 2:]  # the timed step (warm-up and timed steps launch the same sequence)
    widths = w.passes()
    ebs = w.pass_elem_bytes()
    kinds = w.lean_pass_views()
    with open(log + ".views.json") as f:  # (train rows, their nnz, nnz into train rows) per partition
        views = json.load(f)
    self_term = {"gcn": 1, "gin": 1, "sage": 0}[w.model]
    passes, cur = [], None
    for d in seq:
        if ("agg_fixup" in d["kernel"] or "exact_fix" in d["kernel"]) and cur is not None:
            cur["time_us"] += d["gpu__time_duration.sum"]
            cur["dram_bytes"] += d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
            cur["l2_bytes"] += d["lts__t_bytes.sum"]
            cur["fixups"] += 1
            continue
        i = len(passes)
        part, pi = i // len(widths), i % len(widths)
        width, eb = widths[pi], ebs[pi]
        nnz, rows = meta["part_nnz"][part], meta["part_rows"][part]
        rows_in = rows
        if kinds[pi] == "train_rows":  # the lean train step's views (gnn.cu forward / backward(lean))
            rows, nnz = views[part][0], views[part][1]
        elif kinds[pi] == "train_nbrs":
            nnz = views[part][2]
        cur = {"partition": part, "pass": pi, "width": width, "elem_bytes": eb, "kernel": d["kernel"],
               "view": kinds[pi], "nnz": nnz, "rows": rows,
               "time_us": d["gpu__time_duration.sum"],
               "dram_bytes": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
               "dram_read": d["dram__bytes_read.sum"], "dram_write": d["dram__bytes_write.sum"],
               "l2_bytes": d["lts__t_bytes.sum"], "l2_hit_pct": d["lts__t_sector_hit_rate.pct"],
               "l1_hit_pct": d["l1tex__t_sector_hit_rate.pct"], "fixups": 0,
               "algorithmic_bytes": nnz * (4 + eb * width) + rows * (eb * width * self_term + 4 * width + 8),
               "compulsory_bytes": compulsory_bytes(nnz, rows_in, rows, width, eb)}
        passes.append(cur)
    assert len(passes) == w.partitions * len(widths), (len(passes), w.partitions, widths)
    tot = {k: sum(p[k] for p in passes) for k in ("time_us", "dram_bytes", "l2_bytes", "algorithmic_bytes",
                                                  "compulsory_bytes")}
    by_width = {}
    for p in passes:
        b = by_width.setdefault(f'{p["width"]} {"f16" if p["elem_bytes"] == 2 else "f32"}', {"launches": 0, "time_us": 0.0, "dram_bytes": 0.0,
                                                  "algorithmic_bytes": 0.0, "compulsory_bytes": 0.0})
        b["launches"] += 1
        for k in ("time_us", "dram_bytes", "algorithmic_bytes", "compulsory_bytes"):
            b[k] += p[k]
    res = {"workload": workload, "workload_key": w.key(),
           "source": "ncu --metrics " + ",".join(METRICS) + " --clock-control none -k regex:agg_ "
                     "(scripts/k2_traffic.py): every K2 launch of one eager bench step (all partitions, all "
                     "passes; split-row fix-ups and the guard's exact-fix kernels folded into their pass)",
           "passes_per_step": len(passes), "per_step": tot,
           "dram_bytes_per_launch": tot["dram_bytes"] / len(passes),
           "traffic_over_compulsory": tot["dram_bytes"] / tot["compulsory_bytes"],
           "ncu_dram_gbs": tot["dram_bytes"] / (tot["time_us"] * 1e3), "by_width": by_width, "launches": passes}
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "launches"}))


if __name__ == "__main__":
    main()
