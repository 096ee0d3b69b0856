#!/bin/bash
# fast hand-off between update items (next item's first ring groups loaded in the
# current item's last panels, no dependency spin / ring re-init) + C1 rows added
# after step A.  Parity subset, then same-box A/B: new / nofast (C1-late only) / base (HEAD)
OUT=gpurun_out/r02ag
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
for r in 1 2 3; do
  for v in new nofast base; do
    if [ $v = new ]; then L=paper_1102_5328_b200/libtileqr.so; else L=paper_1102_5328_b200/libtileqr_$v.so; fi
    echo "== $v"
    TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16
    TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --n 2048 --pairs 64:16
  done
done > $OUT/ab.log 2>&1
echo done
