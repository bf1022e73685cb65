#!/bin/bash
# A/B of library variants built under paper_2604_15186_b200/lib/<name>/ (build.build(out=...)):
#   VARIANTS="v_a v_b" ENVS="ALP_U_BPS=23" bash tools/ab_variants.sh
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS}; do
for e in ${ENVS:-NONE=1}; do
  env ALP_LIB=paper_2604_15186_b200/lib/$v/libscepsy_alp.so $e python bench.py --workload ${WL:-C4} --steps ${STEPS:-200} --warmup 5 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v $e step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],4), 'idx', d['result']['index'])"
done; done; done
