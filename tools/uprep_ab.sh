for v in v_f3 v_s8 v_s16; do for th in 256 512 1024; do
  r=$(ALP_UPREP_THREADS=$th ALP_LIB=paper_2604_15186_b200/lib/$v/libscepsy_alp.so SHARD_MODE=nccl python tools/block_hist.py C4 8 0 2>&1 | grep -E "k_uprep us" | tail -1)
  echo "$v thr $th: $r"
done; done
for v in v_f3 v_s8 v_s16; do ALP_LIB=paper_2604_15186_b200/lib/$v/libscepsy_alp.so SHARD_MODE=nccl python tools/shard_timing.py C4 8 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['kernel_ms_max'], d['step_ms_max'])"; done
