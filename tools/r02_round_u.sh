#!/bin/bash
OUT=gpurun_out/r02u
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_factor.py -x -q -p no:cacheprovider -k "not config3 and not config4" > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
for r in 1 2 3; do
  echo "hl2"; python tools/perf_scan.py --n 2048 10000 --pairs 64:16,128:16,64:32 ; python tools/perf_scan.py --panel --n --pairs 64:16,128:16
  echo "hl1"; TILEQR_LIB=paper_1102_5328_b200/libtileqr_hl1.so python tools/perf_scan.py --n 2048 10000 --pairs 64:16,128:16,64:32; TILEQR_LIB=paper_1102_5328_b200/libtileqr_hl1.so python tools/perf_scan.py --panel --n --pairs 64:16,128:16
done > $OUT/ab.log 2>&1
