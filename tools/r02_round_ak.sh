#!/bin/bash
# ncu source-level (SASS) stall sampling of the dataflow kernel, 10000^2 (128, 16):
# one CTA per SM (one warp per SMSP: what a single update warp loses) and the default two
OUT=gpurun_out/r02ak
mkdir -p $OUT
for g in 148 0; do
  name=dag_g$g
  if [ $g = 0 ]; then unset TILEQR_DAG_GRID; else export TILEQR_DAG_GRID=$g; fi
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:dag_kernel -s 1 -c 1 \
    -o $OUT/$name -f python tools/perf_scan.py --n 10000 --pairs 128:16 > $OUT/$name.ncu.log 2>&1
  echo "$name rc=$?" >> $OUT/status.txt
  ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/$name.raw.csv 2>/dev/null
  ncu -i $OUT/$name.ncu-rep --page source --csv > $OUT/$name.source.csv 2>/dev/null
  gzip -f $OUT/$name.source.csv
  rm -f $OUT/$name.ncu-rep
done
echo done
