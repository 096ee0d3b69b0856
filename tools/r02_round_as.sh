#!/bin/bash
# C2 early store (last panel's step C in row-block groups, each group stored
# after its last DMMA): parity of the variant, same-box A/B es / base
OUT=gpurun_out/r02as
mkdir -p $OUT
E=paper_1102_5328_b200/libtileqr_es.so
B=paper_1102_5328_b200/libtileqr.so
TILEQR_LIB=$E timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider -k "not config4 and not config3_full" > $OUT/t_es.log 2>&1; echo "rc=$?" >> $OUT/t_es.log
for r in 1 2 3; do
  for v in es base; do
    if [ $v = es ]; then L=$E; else L=$B; fi
    echo "== $v"
    TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16,128:32
    TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --n 2048 --pairs 64:16
  done
done > $OUT/ab.log 2>&1
python tools/ab_table.py $OUT/ab.log > $OUT/ab_table.txt 2>&1
echo done
