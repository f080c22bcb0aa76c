#!/bin/bash
# Profiling recipe (B200_PROFILING.md) for the bench workload; outputs under gpurun_out/.
#   scripts/profile.sh [K2 launches to capture] [K3 launches to capture]
set -x
export CATGNN_CACHE=${CATGNN_CACHE:-/tmp/catgnn_cache}
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --graph 0 --lanes 1"
NK2=${1:-4}
NK3=${2:-5}
python bench.py $ARGS > /dev/null 2> gpurun_out/prep.err   # build the cache
ncu --metrics gpu__time_duration.sum --clock-control none -c 1000 --csv --log-file gpurun_out/launches.csv \
    python bench.py $ARGS > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:agg_ -s 0 -c $NK2 \
    -o gpurun_out/prof_k2 -f python bench.py $ARGS > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 0 -c $NK3 \
    -o gpurun_out/prof_k3 -f python bench.py $ARGS > /dev/null 2>&1
ls -la gpurun_out/
