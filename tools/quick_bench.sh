#!/bin/bash
# Quick A/B measurement (one GPU): GPU parity tests + C4/C3 bench lines without the CPU leg.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -2 gpurun_out/pytest_gpu.txt
for w in ${WORKLOADS:-C4 C3}; do
  timeout 600 python bench.py --workload $w --steps ${STEPS:-100} --warmup 5 --e2e-steps 2 --no-cpu-baseline > gpurun_out/qb_$w.json 2> gpurun_out/qb_$w.err
  python - "$w" <<'PY'
import json, sys
w = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/qb_{w}.json").read().strip().splitlines()[-1])
except Exception as e:
    print(w, "FAILED", e); print(open(f"gpurun_out/qb_{w}.err").read()[-2000:]); sys.exit()
r = d["roofline"]
print(f"{w} k2_ms {r['kernel_ms']:.4f} frac {r['frac']:.4f} step_ms {d['ms_per_step']:.4f} e2e_ms {d['e2e']['ms_per_step']:.4f} "
      f"idx {d['result']['index']} cnt {d['result']['feasible_count']} clk {d['clocks']['sm_mhz']}")
PY
done
