#!/bin/bash
# A/B runs on the GPU box: K2/K3 parity tests, then bench variants (no e2e / cpu legs).
#   scripts/ab.sh "ENV=1 ENV2=3" "ENV=0" ...
timeout 400 python -m pytest tests/test_gpu_sgc.py tests/test_gpu_gemm.py tests/test_gpu_gnn.py -x -q 2>&1 | tail -3
for v in "$@"; do
  echo "== $v"
  env $v timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; g=d['gemm']; print(f\"value {d['value']/1e9:.2f} Ge/s  ms/step {d['ms_per_step']:.2f}  agg {r['agg_ms_per_step']:.2f} ms  gemm {g['ms_per_step']:.2f} ms  launches {d['gpu_launches']}\")"
done
