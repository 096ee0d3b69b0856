#!/bin/bash
# panel step chain A/B: libtileqr.so (split-group reduction + one-step refinements),
# _old (round-1 step: xor fold + two Newton steps each), _xor (xor fold, new scalar chain)
OUT=gpurun_out/r02y
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_factor.py tests/test_gpu_tree.py -x -q -p no:cacheprovider -k "not config3 and not config4" > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
TILEQR_LIB=paper_1102_5328_b200/libtileqr_prof.so timeout 300 python tools/panel_prof.py > $OUT/pprof.log 2>&1
for r in 1 2 3; do
  for v in new old xor; do
    if [ $v = new ]; then L=paper_1102_5328_b200/libtileqr.so; else L=paper_1102_5328_b200/libtileqr_$v.so; fi
    echo "== $v"
    TILEQR_LIB=$L python tools/perf_scan.py --n 2048 4096 10000 --pairs 64:16,128:16,64:32
    TILEQR_LIB=$L python tools/perf_scan.py --panel --n --pairs 64:16,128:16,128:32,256:16,64:8
  done
done > $OUT/ab.log 2>&1
echo done
