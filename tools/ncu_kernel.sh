#!/bin/bash
# One full ncu capture (source-level SASS counts) of the search kernel of one workload:
#   bash tools/ncu_kernel.sh C3 prof_C3 [kernel-regex]
# -> gpurun_out/<name>.ncu-rep ; read here with
#   ncu -i gpurun_out/<name>.ncu-rep --page source --csv --print-source sass > x.csv
#   python tools/sass_blocks.py x.csv --candidates N
W=${1:-C4}; NAME=${2:-prof_$W}; K=${3:-regex:k_search}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "$K" -s 3 -c 1 -f -o gpurun_out/$NAME \
   python bench.py --workload $W --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/$NAME.txt 2>&1
echo "ncu rc=$?"
