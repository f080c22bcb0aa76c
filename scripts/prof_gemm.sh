#!/bin/bash
export CATGNN_CACHE=${CATGNN_CACHE:-/tmp/catgnn_cache}
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > /dev/null 2>&1   # build the cache
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gemm -c 20 --csv --log-file gpurun_out/gemm_launches.csv python bench.py $ARGS > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 0 -c 5 -o gpurun_out/prof_k3b -f python bench.py $ARGS > /dev/null 2>&1
ls -la gpurun_out
