(timeout 1500 python tests/sweep_parity.py 700 90000 | tail -3
 ALP_NO_UR=1 timeout 1200 python tests/sweep_parity.py 300 91000 | tail -3
 ALP_NO_FUSED=1 timeout 1200 python tests/sweep_parity.py 300 92000 | tail -3) > gpurun_out/parity_sweep.txt 2>&1
tail -12 gpurun_out/parity_sweep.txt
