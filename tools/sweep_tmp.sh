for i in 1 2; do for cfg in "12 0" "10 0" "10 2"; do
  set -- $cfg
  if [ $2 = 0 ]; then unset ALP_BLOCKS_PER_SM; else export ALP_BLOCKS_PER_SM=$2; fi
  ALP_ROWS_PER_LANE=$1 timeout 300 python bench.py --workload C4 --steps 100 --warmup 5 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('T=$1 MB=$2', 'k', round(d['roofline']['kernel_ms'],4), 'step', round(d['ms_per_step'],4), d['result']['index'], d['result']['feasible_count'])"
done; done
