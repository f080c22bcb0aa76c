# ncu --set full of the first partition's four K2 passes and the bench launch list.
set -x
mkdir -p gpurun_out
export CATGNN_CACHE=/tmp/catgnn_cache
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --graph 0"
python bench.py $ARGS > /dev/null 2> gpurun_out/prep.err
ncu --set full --clock-control none --import-source on -k regex:agg_kernel -s 0 -c 4 \
    -o gpurun_out/r02_prof_k2 -f python bench.py $ARGS > gpurun_out/ncu_k2.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r02_launches.csv \
    python bench.py $ARGS > /dev/null 2>&1
ls -la gpurun_out
