#!/bin/bash
# Tuning sweep (one GPU): kernel ms with the warp-uniform (constant-bank) path on/off, C4 and C3.
mkdir -p gpurun_out
for w in C4 C3; do
for u in 1 0; do
  ALP_UNIFORM=$u timeout 300 python bench.py --workload $w --steps 30 --warmup 3 --e2e-steps 2 --no-cpu-baseline > gpurun_out/sweep_${w}_u$u.json 2>gpurun_out/sweep_${w}_u$u.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_${w}_u$u.json')); print('$w uniform=$u', 'kernel_ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3), 'step_ms', round(d['ms_per_step'],4), 'launches', d['gpu_launches'], 'idx', d['result']['index'], 'cnt', d['result']['feasible_count'])" || tail -3 gpurun_out/sweep_${w}_u$u.err
done; done
