timeout 600 python -m pytest tests/test_budget_sweep.py tests/test_gpu_parity.py -q -x -k "budget or egalitarian or sweep" 2>&1 | tail -2
python tools/budget_sweep_timing.py 64
ALP_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/bench_2rank_auto.json 2> gpurun_out/bench_2rank_auto.err; echo "auto rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench_2rank_auto.json').read().strip().splitlines()[-1]); print(d['config']['parallelism'], d['config'].get('exchange_probe'), d['value'], d['result']['index'])"
tail -3 gpurun_out/bench_2rank_auto.err
