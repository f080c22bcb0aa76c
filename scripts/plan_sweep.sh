#!/bin/bash
# K2 work-plan sweep (unit cost U x per-row cost) on three reddit partitions.
for u in 256 512 1024; do for rc in 8 16 32; do
  for P in 0 3 7; do
    echo -n "U=$u rc=$rc P=$P "
    CATGNN_UNIT=$u CATGNN_ROW_COST=$rc PART=$P WIDTHS=256,48 REPS=5 python scripts/agg_micro.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read())['k2']; print(d['256']['us'], d['48']['us'])"
  done
done; done
