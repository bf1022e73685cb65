for i in 1 2; do
ALP_U_GSPLIT=1 python tools/step_timeline.py --mode search 2>&1 | grep -v -i warn | head -4
ALP_U_GSPLIT=1 ALP_U_GNOEV=1 python tools/step_timeline.py --mode search 2>&1 | grep -v -i warn | head -4
done
ALP_U_GSPLIT=1 WORKLOADS="C4" PYTEST_ARGS="-k nothing_selected_xyz" bash tools/quick_bench.sh | tail -1
WORKLOADS="C4" PYTEST_ARGS="-k nothing_selected_xyz" bash tools/quick_bench.sh | tail -1
