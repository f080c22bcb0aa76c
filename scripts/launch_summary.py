"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel."""
import csv
import re
import sys
from collections import defaultdict

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = [r for r in csv.DictReader(lines) if r.get("Metric Name") == "gpu__time_duration.sum"]
agg = defaultdict(lambda: [0, 0.0])
for r in rows:
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").replace("catgnn::", "")
    name = name.replace("<unnamed>::", "")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    v = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)  # -> usecond
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'n':>5s} {'total ms':>9s} {'share':>6s} {'us/launch':>9s}")
for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {n:5d} {t / 1e3:9.3f} {100 * t / tot:5.1f}% {t / n:9.1f}")
print(f"total {tot / 1e3:.3f} ms over {sum(v[0] for v in agg.values())} launches")
