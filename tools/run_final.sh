#!/bin/bash
# Round-end measurement set (one GPU): tests, smoke, bench lines (C4 headline with CPU oracle leg,
# C3, C5, reference arm), device timeline, per-rank shard timing (NCCL-path and peer-exchange
# modes), budget-sweep timing, 2-rank gloo path (NCCL exchange and peer exchange), ncu launch list
# and full ncu captures of the search kernel on C4 and C3.  Then: bash tools/collect_profiles.sh r02
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu_info.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)|Socket|Core" > gpurun_out/host_cpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 600 python bench.py > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err
timeout 600 python bench.py --workload C3 --steps 50 --warmup 3 --e2e-steps 3 --cpu-seconds 20 > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err
timeout 600 python bench.py --workload C5 --steps 5 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
python tools/step_timeline.py --workload C4 --mode search > gpurun_out/timeline_C4_search.txt 2>/dev/null
python tools/step_timeline.py --workload C4 --mode shard > gpurun_out/timeline_C4_shard.txt 2>/dev/null
python tools/step_timeline.py --workload C4 --mode peer > gpurun_out/timeline_C4_peer.txt 2>/dev/null
(for m in nccl peer; do SHARD_MODE=$m python tools/shard_timing.py C4; done; SHARD_MODE=nccl python tools/shard_timing.py C3) > gpurun_out/shard_timing.jsonl 2>&1
(for w in "C4 8 0" "C4 1 0"; do for m in nccl peer; do SHARD_MODE=$m python tools/block_hist.py $w 2>&1 | grep -E "^\[|peer epi|finalize \(|tickets|histogram"; done; done) > gpurun_out/block_timeline_C4.txt
(python tools/budget_sweep_timing.py 64; ALP_NO_LEVELS=1 python tools/budget_sweep_timing.py 64) > gpurun_out/budget_sweep.jsonl 2>&1
bash tools/multirank_check.sh > gpurun_out/multirank.txt 2>&1
ALP_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 20 --warmup 3 --e2e-steps 2 --exchange peer > gpurun_out/bench_2rank_peer.json 2> gpurun_out/bench_2rank_peer.err
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launch_bench.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_search -s 3 -c 1 -f -o gpurun_out/prof_search \
   python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_search -s 3 -c 1 -f -o gpurun_out/prof_search_C3 \
   python bench.py --workload C3 --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_full_C3.txt 2>&1
fi
tail -2 gpurun_out/pytest_gpu.txt; cat gpurun_out/smoke.txt; head -c 400 gpurun_out/bench_C4.json; echo
