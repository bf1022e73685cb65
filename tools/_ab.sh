for i in 1 2; do
for v in cur old; do
  L=""; [ $v = old ] && L="ALP_LIB=paper_2604_15186_b200/lib/variant_old/libscepsy_alp.so"
  env $L python bench.py --steps 100 --warmup 5 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],4))"
  env $L SHARD_MODE=nccl python tools/shard_timing.py C4 1,8 20 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print('$v shard world',d['world'],'kmax %.4f smax %.4f'%(d['kernel_ms_max'],d['step_ms_max']))"
done; done
python tools/step_timeline.py --workload C4 --mode shard 2>/dev/null | head -6
ALP_DBG_TS=1 python tools/shard_timing.py C4 1 3 2>&1 | grep "k_uprep us" | tail -2
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
