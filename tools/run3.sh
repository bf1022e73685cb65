bash tools/variant_sweep.sh > gpurun_out/sweep.txt 2>&1
NCU=0 bash tools/gpu_check.sh
