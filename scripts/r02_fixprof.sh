set -x
export CATGNN_CACHE=/tmp/catgnn_cache
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline --graph 0"
CATGNN_GUARD_STATS=1 python bench.py $ARGS 2>&1 >/dev/null | grep guard | tail -8
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:exact_fix -c 4 python bench.py $ARGS 2>&1 | grep -E "exact_fix|duration|dram__|lts__|warps_active|inst_exec" | head -40
