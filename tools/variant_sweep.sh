#!/bin/bash
# Tuning sweep (one GPU): kernel ms per (rows per lane, blocks per SM) on C4 and C3.
mkdir -p gpurun_out
for w in C4 C3; do
for cfg in "8 3" "8 4" "16 2" "16 3"; do
  set -- $cfg
  ALP_ROWS_PER_LANE=$1 ALP_BLOCKS_PER_SM=$2 timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/sweep_${w}_t$1_b$2.json 2>gpurun_out/sweep_${w}_t$1_b$2.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_${w}_t$1_b$2.json')); print('$w T=$1 MB=$2', 'kernel_ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3), 'step_ms', round(d['ms_per_step'],4), 'idx', d['result']['index'], 'cnt', d['result']['feasible_count'])" || tail -3 gpurun_out/sweep_${w}_t$1_b$2.err
done; done
