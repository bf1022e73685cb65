#!/bin/bash
# Kernel-variant sweep: kernel ms per inner-loop encoding on C4 and C3 (one GPU).
mkdir -p gpurun_out
for w in C4 C3; do
for v in 0 1 2 3; do
  ALP_KERNEL_VARIANT=$v timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sweep_${w}_v$v.json 2>gpurun_out/sweep_${w}_v$v.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_${w}_v$v.json')); print('$w v$v', 'kernel_ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3), 'step_ms', round(d['ms_per_step'],4), 'idx', d['result']['index'], 'cnt', d['result']['feasible_count'])" || tail -3 gpurun_out/sweep_${w}_v$v.err
done; done
