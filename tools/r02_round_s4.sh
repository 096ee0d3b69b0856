#!/bin/bash
# session 4: resident-CTA count of the dataflow kernel at small N (panel-latency bound sizes)
OUT=gpurun_out/r02s4_grid.log
: > $OUT
for n in 1000 2048 4000; do
for g in 296 222 148 74; do
  printf "n=%s grid=%s " $n $g >> $OUT
  TILEQR_DAG_GRID=$g python tools/perf_scan.py --n $n --pairs 64:16,64:32 2>/dev/null | tr '\n' ' ' >> $OUT
  echo >> $OUT
done
done
for s in 3000,3000,5000 1500,1500,5000 1500,1500,2000 3000,3000,2000 5000,5000,5000; do
  printf "n=2048 sim=%s " $s >> $OUT
  TILEQR_DAG_SIM=$s python tools/perf_scan.py --n 2048 --pairs 64:16 2>/dev/null | tr '\n' ' ' >> $OUT
  echo >> $OUT
done
cat $OUT
