#!/bin/bash
# session 4: tail retirement (second CTA of each SM stops claiming in the list's tail) -- sweep of the tail length
OUT=gpurun_out/r02s4_retire.log
: > $OUT
timeout 300 python -m pytest tests/test_gpu_factor.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2 >> $OUT
for n in 10000 6000; do
for r in 0 3000 8000 15000 30000 0 8000; do
  printf "n=%s retire=%s " $n $r >> $OUT
  TILEQR_DAG_RETIRE=$r timeout 120 python tools/perf_scan.py --n $n --pairs 128:16,128:32 2>/dev/null | cut -c1-90 | tr '\n' ' ' >> $OUT
  echo >> $OUT
done
done
printf "tests with retire=8000: " >> $OUT
TILEQR_DAG_RETIRE=8000 timeout 300 python -m pytest tests/test_gpu_factor.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -1 >> $OUT
cat $OUT
