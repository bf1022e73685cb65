#!/bin/bash
# Slowest-rank shard step at 8 ranks for shard-range cost weights (ALP_SHARD_PARTIAL / ALP_SHARD_MIXED).
for p in 1 1.0625 1.125 1.1875 1.25; do for m in ${MIXED:-1.375}; do
  ALP_SHARD_PARTIAL=$p ALP_SHARD_MIXED=$m SHARD_MODE=nccl python tools/shard_timing.py ${WL:-C4} 8 20 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('partial $p mixed $m: kernel max %.4f step max %.4f slowest %d' % (d['kernel_ms_max'], d['step_ms_max'], d['slowest_rank']))"
done; done
