#!/bin/bash
# C2 loads row blocks outer (panel-0 step A order)
OUT=gpurun_out/r02av
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_parity.py tests/test_gpu_dist.py tests/test_gpu_tree.py -x -q -p no:cacheprovider -k "not config4" > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
for r in 1 2 3; do
  for v in new prev; do
    if [ $v = new ]; then L=paper_1102_5328_b200/libtileqr.so; else L=paper_1102_5328_b200/libtileqr_$v.so; fi
    echo "== $v"
    TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16,128:32
    TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --n 20000 --pairs 160:16
  done
done > $OUT/ab.log 2>&1
python tools/ab_table.py $OUT/ab.log > $OUT/ab_table.txt 2>&1
echo done
