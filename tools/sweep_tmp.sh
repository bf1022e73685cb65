for cfg in "C4 8 lib" "C4 16 lib" "C4 16 u1" "C4 8 u1" "C3 16 lib" "C3 16 u1"; do
  set -- $cfg
  if [ $3 = u1 ]; then export ALP_LIB=paper_2604_15186_b200/lib/v_u1.so; else unset ALP_LIB; fi
  ALP_ROWS_PER_LANE=$2 timeout 300 python bench.py --workload $1 --steps 50 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('$cfg', 'k2', round(d['roofline']['kernel_ms'],4), 'frac', round(d['roofline']['frac'],3), 'idx', d['result']['index'], 'cnt', d['result']['feasible_count'])" || tail -3 gpurun_out/sw.err
done
