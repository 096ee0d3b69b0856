#!/bin/bash
# early store default (ES = 4, NB >= 96): full GPU suite on the default lib,
# same-box A/B default / es2 / base (no early store)
OUT=gpurun_out/r02at
mkdir -p $OUT
for r in 1 2 3; do
  for v in new es2 base; do
    if [ $v = new ]; then L=paper_1102_5328_b200/libtileqr.so; else L=paper_1102_5328_b200/libtileqr_$v.so; fi
    echo "== $v"
    TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16,128:32
    TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --n 20000 --pairs 256:32,160:16
  done
done > $OUT/ab.log 2>&1
python tools/ab_table.py $OUT/ab.log > $OUT/ab_table.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gpu_tests.txt 2>&1; echo "rc=$?" >> $OUT/gpu_tests.txt
echo done
