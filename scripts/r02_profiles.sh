# profiles only (one stream): K2 traffic of all passes, ncu --set full of partition 0's K2 passes,
# exact fix and first K3 launches, launch list
set -x
mkdir -p gpurun_out
export CATGNN_CACHE=/tmp/catgnn_cache
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --graph 0 --lanes 1"
python bench.py $ARGS > /dev/null 2> gpurun_out/prep.err
timeout 900 python scripts/k2_traffic.py reddit_gcn gpurun_out/r02_k2_traffic_reddit_gcn.json > gpurun_out/k2t.log 2>&1
tail -c 600 gpurun_out/k2t.log
ncu --set full --clock-control none --import-source on -k regex:agg_kernel -s 0 -c 4 \
    -o gpurun_out/r02_k2_full -f python bench.py $ARGS > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:exact_fix -s 0 -c 2 \
    -o gpurun_out/r02_fix_full -f python bench.py $ARGS > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tf32 -s 0 -c 5 \
    -o gpurun_out/r02_k3_full -f python bench.py $ARGS > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py $ARGS > /dev/null 2>&1
ls -la gpurun_out | tail -8
