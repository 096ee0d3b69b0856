#!/bin/bash
# row-limited SSRFB out of line (noinline, no hook); 8-warp / MB=1 CTA variant (w8) for NB=128:
# parity subset on the default lib, w8 parity on the factor tests, same-box A/B new / w8 / base
OUT=gpurun_out/r02al
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
W=paper_1102_5328_b200/libtileqr_w8.so
B=paper_1102_5328_b200/libtileqr_base.so
TILEQR_LIB=$W timeout 900 python -m pytest tests/test_gpu_factor.py -x -q -p no:cacheprovider -k "not config4" > $OUT/t_w8.log 2>&1; echo "rc=$?" >> $OUT/t_w8.log
for r in 1 2; do
  for v in new w8 base; do
    if [ $v = new ]; then L=paper_1102_5328_b200/libtileqr.so; elif [ $v = w8 ]; then L=$W; else L=$B; fi
    echo "== $v"
    TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16,128:32
    TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --n 2048 --pairs 64:16,96:32
  done
done > $OUT/ab.log 2>&1
TILEQR_LIB=$W timeout 600 python tools/trace_factor.py --n 10000 --nb 128 --ib 16 --out $OUT/trace_w8.json > $OUT/trace_w8.log 2>&1
python tools/trace_sm.py $OUT/trace_w8.json > $OUT/trace_w8_sm.txt 2>&1; rm -f $OUT/trace_w8.json
echo done
