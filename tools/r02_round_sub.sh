#!/bin/bash
# sub-task width A/B (TILEQR_PANEL_SUB: columns per GEQRT/TSQRT sub-task of the DAG)
OUT=gpurun_out/r02ad
mkdir -p $OUT
for r in 1 2 3; do
  for sc in 32 16 64 128; do
    echo "== sc$sc"
    TILEQR_PANEL_SUB=$sc python tools/perf_scan.py --n 1024 2048 4096 --pairs 64:16,128:16,64:8,128:32
    TILEQR_PANEL_SUB=$sc python tools/perf_scan.py --n 10000 --pairs 128:16
  done
done > $OUT/ab.log 2>&1
echo done
