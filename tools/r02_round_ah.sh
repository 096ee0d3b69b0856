#!/bin/bash
# fast hand-off (C1 seeded as before) + SSRFB row limit on the padded tile row +
# claim-ahead window: parity subset, then same-box A/B against base (HEAD) and env variants
OUT=gpurun_out/r02ah
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_parity.py tests/test_gpu_dist.py -x -q -p no:cacheprovider > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
B=paper_1102_5328_b200/libtileqr_base.so
for r in 1 2; do
  echo "== new"; timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16
  echo "== norowlim"; TILEQR_DAG_NO_ROWLIM=1 timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16
  for t in 300 900 2000; do echo "== tail$t"; TILEQR_DAG_CA_TAIL=$t timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16; done
  for h in 300 1500; do echo "== head$h"; TILEQR_DAG_CA_HEAD=$h timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16; done
  echo "== base"; TILEQR_LIB=$B timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16
done > $OUT/ab.log 2>&1
for r in 1 2; do
  echo "== new"; timeout 300 python tools/perf_scan.py --n 2048 --pairs 64:16
  for t in 100 300; do echo "== tail$t"; TILEQR_DAG_CA_TAIL=$t timeout 300 python tools/perf_scan.py --n 2048 --pairs 64:16; done
  echo "== base"; TILEQR_LIB=$B timeout 300 python tools/perf_scan.py --n 2048 --pairs 64:16
done > $OUT/ab2048.log 2>&1
echo done
