#!/bin/bash
# Copy the outputs of tools/run_final.sh (gpurun_out/) into profiles/ under the round prefix.
set -e
R=${1:-r02}
G=gpurun_out
cp $G/bench_C4.json profiles/${R}_bench_C4.json
cp $G/bench_C3.json profiles/${R}_bench_C3.json
cp $G/bench_C5.json profiles/${R}_bench_C5.json
cp $G/bench_reference.json profiles/${R}_bench_reference.json
cp $G/bench_2rank_gloo.json profiles/${R}_bench_C4_2rank_gloo_1gpu.json
cp $G/bench_2rank_peer.json profiles/${R}_bench_C4_2rank_peer_1gpu.json
cp $G/budget_sweep.jsonl profiles/${R}_budget_sweep_timing.jsonl
cp $G/block_timeline_C4.txt profiles/${R}_block_timeline_C4.txt
cp $G/launches.csv profiles/${R}_C4_launches.csv
ncu -i $G/prof_search.ncu-rep --page raw --csv > profiles/${R}_C4_k_search_ncu_raw.csv 2>/dev/null
ncu -i $G/prof_search_C3.ncu-rep --page raw --csv > profiles/${R}_C3_k_search_ncu_raw.csv 2>/dev/null
ncu -i $G/prof_search.ncu-rep --page source --csv --print-source sass > $G/sass_C4.csv 2>/dev/null
python tools/sass_blocks.py $G/sass_C4.csv --candidates 11019960576 --top 30 > profiles/${R}_C4_k_search_sass_blocks.txt
(echo "# fused single-GPU search (alp_search): one kernel, zero-copy result"; cat $G/timeline_C4_search.txt; echo
 echo "# shard path (alp_search_shard + alp_finalize), world 1, no all-reduce; K3 writes the result zero-copy"
 cat $G/timeline_C4_shard.txt; echo
 echo "# peer path (alp_search_peer), one rank over the whole range: search + in-kernel exchange, result zero-copy"
 cat $G/timeline_C4_peer.txt) > profiles/${R}_step_timeline_C4.txt
cp $G/shard_timing.jsonl profiles/${R}_shard_scaling.jsonl
cp $G/pytest_gpu.txt profiles/${R}_pytest_gpu.txt
python tools/ncu_summary.py C4=profiles/${R}_C4_k_search_ncu_raw.csv C3=profiles/${R}_C3_k_search_ncu_raw.csv
