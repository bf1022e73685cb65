#!/bin/bash
# 2 ranks sharing the single GPU over gloo: exercises the sharded search + all-reduce + finalize path.
mkdir -p gpurun_out
ALP_DIST_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 --e2e-steps 2 > gpurun_out/bench_2rank_gloo.json 2> gpurun_out/bench_2rank_gloo.err
echo "2-rank rc=$?"; cat gpurun_out/bench_2rank_gloo.json; tail -3 gpurun_out/bench_2rank_gloo.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference.json 2>gpurun_out/bench_reference.err; echo "ref rc=$?"; cat gpurun_out/bench_reference.json
