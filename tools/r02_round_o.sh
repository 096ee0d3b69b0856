#!/bin/bash
# GPU call: release-RED completion vs fence + atomic (same box), plus dataflow correctness tests
OUT=gpurun_out/r02o
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "dataflow or stress or config2 or every_panel" > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
for r in 1 2 3; do
  echo "release"; python tools/perf_scan.py --n 10000 2048 --pairs 128:16,64:16
  echo "fence"; TILEQR_LIB=paper_1102_5328_b200/libtileqr_fence.so python tools/perf_scan.py --n 10000 2048 --pairs 128:16,64:16
done > $OUT/ab.log 2>&1
