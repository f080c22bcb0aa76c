#!/bin/bash
# configs[4]: partition count k x averaging period s on the reddit-shaped graph, one B200
# (all k partitions on one GPU).  One bench line per cell -> gpurun_out/sweep_ks.jsonl.
out=gpurun_out/sweep_ks.jsonl
: > $out
for k in 2 4 8; do
  w=reddit_gcn_p$k; [ $k = 8 ] && w=reddit_gcn
  for s in 1 4 16; do
    python bench.py --workload $w --sync $s --steps 16 --warmup 3 --no-cpu-baseline 2>>gpurun_out/sweep_ks.err \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); d['sweep']={'k':$k,'s':$s}; print(json.dumps(d))" >> $out
  done
done
python - <<'PY'
import json
for l in open("gpurun_out/sweep_ks.jsonl"):
    d = json.loads(l)
    c = d["config"]
    print(d["sweep"], "ms/step %.2f" % d["ms_per_step"], "value %.2f Ge/s" % (d["value"] / 1e9),
          "e2e %.2f" % (d["e2e"]["value"] / 1e9), "RF %.2f" % c["replication_factor"], "sum/max %.2f" % c["sum_over_max_edges"])
PY
