WORKLOADS="C4" bash tools/quick_bench.sh
for cfg in "ALP_U_TAILW=0" "ALP_U_TAILW=1" "ALP_U_TAILW=4" "ALP_U_TAILQ=6" "ALP_U_TAILQ=2"; do echo "== $cfg"; env $cfg WORKLOADS="C4" PYTEST_ARGS="-k nothing_selected_xyz" bash tools/quick_bench.sh | tail -1; done
ALP_DBG_TS=1 python tools/shard_timing.py C4 2>&1 | grep "alp dbg" | awk 'NR%20==10'
python tools/shard_timing.py C4 2>&1 | tail -5
