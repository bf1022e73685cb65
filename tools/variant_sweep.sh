#!/bin/bash
# Tuning sweep (one GPU): a-class path on/off on C4; C3 default.
mkdir -p gpurun_out
for cfg in "C4 1" "C4 0" "C3 1"; do
  set -- $cfg
  ALP_CLASS_PATH=$2 timeout 300 python bench.py --workload $1 --steps 30 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/sweep_$1_c$2.json 2>gpurun_out/sweep_$1_c$2.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_$1_c$2.json')); print('$1 cls=$2', 'kernel_ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3), 'step_ms', round(d['ms_per_step'],4), 'idx', d['result']['index'], 'cnt', d['result']['feasible_count'])" || tail -3 gpurun_out/sweep_$1_c$2.err
done
