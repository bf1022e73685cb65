for i in 1 2; do for nq in 0 2 3; do
  ALP_NQ=$nq timeout 300 python bench.py --workload C4 --steps 100 --warmup 5 --e2e-steps 1 --no-cpu-baseline > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('nQ=$nq', 'k', round(d['roofline']['kernel_ms'],4), 'step', round(d['ms_per_step'],4), d['result']['index'], d['result']['feasible_count'])"
done; done
