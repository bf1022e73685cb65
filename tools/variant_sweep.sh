#!/bin/bash
# Tuning sweep (one GPU): kernel ms per (rows per lane, blocks per SM) on C4 and C3.
mkdir -p gpurun_out
for w in C4 C3; do
for cfg in "8 3" "8 4" "16 2"; do
  set -- $cfg
  ALP_ROWS_PER_LANE=$1 ALP_BLOCKS_PER_SM=$2 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/sweep_${w}_t$1_b$2.json 2>gpurun_out/sweep_${w}_t$1_b$2.err
  python -c "import json,sys; d=json.load(open('gpurun_out/sweep_${w}_t$1_b$2.json')); print('$w T=$1 MB=$2', 'kernel_ms', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3), 'step_ms', round(d['ms_per_step'],4), 'e2e', '%.3g'%d['e2e']['value'], 'idx', d['result']['index'], 'cnt', d['result']['feasible_count'])" || tail -3 gpurun_out/sweep_${w}_t$1_b$2.err
done; done
ALP_TRACE=1 python - > gpurun_out/trace_build.txt 2>&1 <<'PY'
import time, torch
import paper_2604_15186_b200 as P
from workloads import generate
d = generate.load("C4")
for i in range(4):
    t0 = time.perf_counter(); a = P.Alp.from_instance(d); t1 = time.perf_counter()
    r = a.search(d["targets"][0], d["budget_units"]); t2 = time.perf_counter()
    a.close(); t3 = time.perf_counter()
    print(f"build {1e3*(t1-t0):.3f} ms  search {1e3*(t2-t1):.3f} ms  destroy {1e3*(t3-t2):.3f} ms  kernel {a.last_kernel_ms if False else 0}")
PY
