#!/bin/bash
# panel A/B: libtileqr.so (working tree) vs libtileqr_prev.so (HEAD)
OUT=gpurun_out/r02ac
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_factor.py tests/test_gpu_tree.py -x -q -p no:cacheprovider -k "not config3 and not config4" > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
for r in 1 2 3; do
  for v in new prev; do
    if [ $v = new ]; then L=paper_1102_5328_b200/libtileqr.so; else L=paper_1102_5328_b200/libtileqr_$v.so; fi
    echo "== $v"
    TILEQR_LIB=$L python tools/perf_scan.py --n 2048 4096 10000 --pairs 64:16,128:16,128:32,64:32
    TILEQR_LIB=$L python tools/perf_scan.py --panel --n --pairs 64:16,128:16,128:32,256:16,64:8,96:24
  done
done > $OUT/ab.log 2>&1
echo done
