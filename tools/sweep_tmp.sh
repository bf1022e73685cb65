for cfg in "0 0" "3 0" "3 1" "2 1" "0 0" "3 1"; do
  set -- $cfg
  if [ $2 = 1 ]; then export ALP_ALIGN_GRABS=1; else unset ALP_ALIGN_GRABS; fi
  echo "nQ=$1 align=$2 $(ALP_NQ=$1 python tools/shard_timing.py C4 | python -c "
import sys, json
print(' '.join('w%d:%.4f' % (d['world'], d['kernel_ms']) for d in map(json.loads, sys.stdin)))")"
done
