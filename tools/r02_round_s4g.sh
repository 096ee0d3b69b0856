#!/bin/bash
# session 4: same-box A/B of the build with / without the tail-retirement code at 10000^2 and 6000^2
OUT=gpurun_out/r02s4_retire_build_ab.log
: > $OUT
NORET=$PWD/paper_1102_5328_b200/libtileqr_noret.so
for rep in 1 2 3; do
  printf "noret_build " >> $OUT
  (TILEQR_LIB=$NORET python tools/perf_scan.py --n 10000 --pairs 128:16,128:32; TILEQR_LIB=$NORET python tools/perf_scan.py --n 6000 --pairs 128:16) 2>/dev/null | cut -c7-80 | tr '\n' ' ' >> $OUT; echo >> $OUT
  for t in 500 250; do
    printf "retire_build tiles=%s " $t >> $OUT
    (TILEQR_DAG_RETIRE_TILES=$t python tools/perf_scan.py --n 10000 --pairs 128:16,128:32; TILEQR_DAG_RETIRE_TILES=$t python tools/perf_scan.py --n 6000 --pairs 128:16) 2>/dev/null | cut -c7-80 | tr '\n' ' ' >> $OUT; echo >> $OUT
  done
done
cat $OUT
