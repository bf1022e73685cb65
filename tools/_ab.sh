for i in 1 2; do
for v in cur old; do
  L=""; [ $v = old ] && L="ALP_LIB=paper_2604_15186_b200/lib/variant_old/libscepsy_alp.so"
  env $L python bench.py --steps 100 --warmup 5 --e2e-steps 1 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v step', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done; done
for v in cur old; do
  L=""; [ $v = old ] && L="ALP_LIB=paper_2604_15186_b200/lib/variant_old/libscepsy_alp.so"
  env $L SHARD_MODE=peer python tools/shard_timing.py C4 1,8 20 2>&1 | cut -c1-150 | sed "s/^/$v /"
done
