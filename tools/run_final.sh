#!/bin/bash
# Round-end measurement set (one GPU): tests, smoke, C4 bench (+ ncu), C5 and C3 bench lines.
mkdir -p gpurun_out
bash tools/gpu_check.sh
timeout 600 python bench.py --workload C5 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 600 python bench.py --workload C3 --steps 50 --warmup 3 --e2e-steps 2 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
ALP_TRACE=1 timeout 120 python -c "
import time, sys; sys.path.insert(0, '.')
import paper_2604_15186_b200 as P
from workloads import generate
d = generate.load('C4'); desc = P.Desc(d)
for i in range(5):
    t0 = time.perf_counter(); a = P.Alp.build(desc); t1 = time.perf_counter()
    r = a.search(d['targets'][0], d['budget_units']); t2 = time.perf_counter(); a.close(); t3 = time.perf_counter()
    print(f'build {1e3*(t1-t0):.3f} ms search {1e3*(t2-t1):.3f} ms destroy {1e3*(t3-t2):.3f} ms')
" > gpurun_out/trace_e2e.txt 2>&1
