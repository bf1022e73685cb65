#!/bin/bash
# Tail split candidates at 8 ranks, three repeats each (slowest-rank shard kernel / step).
for r in 1 2 3; do for sp in 0.5,3 0.5,2 0.25,3 0.25,2; do
  ALP_U_SPLIT=$sp SHARD_MODE=nccl python tools/shard_timing.py C4 8 30 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('split $sp rep $r: kmax %.4f smax %.4f' % (d['kernel_ms_max'], d['step_ms_max']))"
done; done
for sp in 0.5,3 0.5,2; do ALP_U_SPLIT=$sp python bench.py --steps 200 --warmup 5 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C4 N=1 split $sp step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4))"; done
