#!/bin/bash
# session 4: one resident CTA per SM for small DAGs -- crossover of the rule (thr 0 = off, 1e9 = always)
OUT=gpurun_out/r02s4_one_cta.log
: > $OUT
for n in 500 1000 1500 2048 2500 3000 3500 4000; do
for thr in 0 1000000000; do
  printf "n=%s thr=%s " $n $thr >> $OUT
  TILEQR_DAG_ONE_CTA_TILES=$thr python tools/perf_scan.py --n $n --pairs 64:16,64:32,128:16 2>/dev/null | cut -c1-90 | tr '\n' ' ' >> $OUT
  echo >> $OUT
done
done
cat $OUT
