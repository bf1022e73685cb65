#!/bin/bash
# Occupancy (ALP_U_BPS) on C3 and tail split (ALP_U_SPLIT=x,S) on C4 at 1 and 8 ranks.
for b in 16 20 24; do
  ALP_U_BPS=$b python bench.py --workload C3 --steps 30 --warmup 3 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C3 bps $b kernel', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],4))"
done
for sp in 0.5,3 0.25,3 1,3 0.5,2 0.5,6 0,1; do
  ALP_U_SPLIT=$sp SHARD_MODE=nccl python tools/shard_timing.py C4 1,8 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('split $sp world', d['world'], 'kmax %.4f smax %.4f' % (d['kernel_ms_max'], d['step_ms_max']))"
done
