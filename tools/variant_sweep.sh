#!/bin/bash
# Tuning sweep: kernel ms per rows-per-lane setting on C4 and C3 (one GPU).
mkdir -p gpurun_out
for w in C4 C3; do
for t in 8 16; do
  ALP_ROWS_PER_LANE=$t timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/sweep_${w}_t$t.json 2>gpurun_out/sweep_${w}_t$t.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_${w}_t$t.json')); print('$w T=$t', 'kernel_ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3), 'step_ms', round(d['ms_per_step'],4), 'e2e', '%.3g'%d['e2e']['value'], 'idx', d['result']['index'], 'cnt', d['result']['feasible_count'])" || tail -3 gpurun_out/sweep_${w}_t$t.err
done; done
