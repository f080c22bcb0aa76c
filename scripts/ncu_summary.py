"""Per-launch metrics from an `ncu --set full` report (ncu -i ... --page raw --csv).

    python scripts/ncu_summary.py REPORT.ncu-rep [--traffic-json OUT --workload NAME]
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "time_us": ("gpu__time_duration.sum", None),
    "dram_read": ("dram__bytes_read.sum", None),
    "dram_write": ("dram__bytes_write.sum", None),
    "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "lts_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "dram_pct": ("dram__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "sm_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "tensor_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "regs": ("launch__registers_per_thread", 1),
    "grid": ("launch__grid_size", 1),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "nsecond": 1e-3, "usecond": 1, "msecond": 1e3, "second": 1e6,
              "ns": 1e-3, "us": 1, "ms": 1e3, "s": 1e6}


def rows(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    head, units = r[0], r[1]
    res = []
    for row in r[2:]:
        d = {"kernel": row[head.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for k, (name, _) in KEYS.items():
            if name in head:
                i = head.index(name)
                try:
                    v = float(row[i].replace(",", ""))
                except ValueError:
                    continue
                d[k] = v * UNIT_SCALE.get(units[i], 1)
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--traffic-json")
    ap.add_argument("--workload", default="reddit_gcn")
    ap.add_argument("--source", default="")
    a = ap.parse_args()
    rs = rows(a.report)
    for d in rs:
        print(json.dumps(d))
    if a.traffic_json:
        # one K2 "launch" in bench.py = an aggregation pass: the main kernel plus its fix-up
        per = [d.get("dram_read", 0) + d.get("dram_write", 0) for d in rs]
        passes = max(1, sum(1 for d in rs if "fixup" not in d["kernel"]))
        json.dump({"workload": a.workload, "source": a.source,
                   "dram_bytes_per_launch": sum(per) / passes, "passes": passes, "launches": rs},
                  open(a.traffic_json, "w"), indent=1)


if __name__ == "__main__":
    main()
