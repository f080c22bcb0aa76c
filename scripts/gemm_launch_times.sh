#!/bin/bash
# usage: gemmprof.sh LIBDIR tag
export CATGNN_CACHE=/tmp/catgnn_cache
CATGNN_LIB=$1/libcatgnn.so ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm_tf32 -c 10 --csv --log-file gpurun_out/g_$2.csv python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --graph 0 > /dev/null 2>&1
python - gpurun_out/g_$2.csv <<'PY'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>5]
h=rows[0]; i=h.index('Metric Value'); k=h.index('Kernel Name')
print(sys.argv[1], [ (r[k][:22], r[i]) for r in rows[1:]])
PY
