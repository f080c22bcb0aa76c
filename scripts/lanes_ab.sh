for cfg in "1 0 0" "2 0 0" "2 116 32" "2 124 24" "2 108 40" "4 116 32" "1 0 0"; do
  set -- $cfg
  timeout 300 python bench.py --no-e2e --no-cpu-baseline --lanes $1 --agg-sms $2 --gemm-sms $3 2>gpurun_out/lanes_err.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lanes=$1 agg=$2 gemm=$3', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/lanes_err.log
done
