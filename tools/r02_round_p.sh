#!/bin/bash
# GPU call: ring carry-over -- correctness first (bounded), then same-box A/B
OUT=gpurun_out/r02p
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_factor.py -x -q -p no:cacheprovider -k "dataflow or stress or host" > $OUT/t1.log 2>&1; echo "rc=$?" >> $OUT/t1.log
if grep -q "rc=0" $OUT/t1.log; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/t_all.log 2>&1; echo "rc=$?" >> $OUT/t_all.log
  for r in 1 2 3; do
    echo "carry"; timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16,128:8,96:16
    echo "nocarry"; TILEQR_LIB=paper_1102_5328_b200/libtileqr_nocarry.so timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16,128:8,96:16
  done > $OUT/ab.log 2>&1
fi
