WORKLOADS="C4 C3" bash tools/quick_bench.sh
ALP_DBG_TS=1 python tools/shard_timing.py C4 2>&1 | grep "alp dbg" | awk 'NR%20==10'
python tools/shard_timing.py C4
