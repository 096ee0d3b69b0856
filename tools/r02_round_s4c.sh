#!/bin/bash
# session 4: one resident CTA per SM -- crossover for NB = 96 / 128 (thr 0 = off, 1e9 = always)
OUT=gpurun_out/r02s4_one_cta_nb128.log
: > $OUT
for n in 2048 3000 4000 5000 6000 8000; do
for thr in 0 1000000000; do
  printf "n=%s thr=%s " $n $thr >> $OUT
  TILEQR_DAG_ONE_CTA_TILES=$thr python tools/perf_scan.py --n $n --pairs 96:16,128:16,128:32 2>/dev/null | cut -c1-90 | tr '\n' ' ' >> $OUT
  echo >> $OUT
done
done
cat $OUT
