#!/bin/bash
# per-inner-panel proxy fence (MEMBAR.ALL.CTA) dropped from the ring release:
# parity subset, same-box A/B new / fence (the fence kept) / base (HEAD), packed SSRFB rates, 1-CTA trace
OUT=gpurun_out/r02aj
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_parity.py tests/test_gpu_kernels.py -x -q -p no:cacheprovider > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
B=paper_1102_5328_b200/libtileqr_base.so
F=paper_1102_5328_b200/libtileqr_fence.so
for r in 1 2; do
  echo "== new"; timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16
  echo "== fence"; TILEQR_LIB=$F timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16
  echo "== base"; TILEQR_LIB=$B timeout 300 python tools/perf_scan.py --n 10000 4096 --pairs 128:16
  echo "== new"; timeout 300 python tools/perf_scan.py --n 2048 --pairs 64:16
  echo "== fence"; TILEQR_LIB=$F timeout 300 python tools/perf_scan.py --n 2048 --pairs 64:16
  echo "== base"; TILEQR_LIB=$B timeout 300 python tools/perf_scan.py --n 2048 --pairs 64:16
done > $OUT/ab.log 2>&1
for v in new base; do
  if [ $v = new ]; then L=paper_1102_5328_b200/libtileqr.so; else L=$B; fi
  echo "== $v"; TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --ssrfb --pairs 128:16,128:32,256:32,64:16,192:32
done > $OUT/ssrfb.log 2>&1
TILEQR_DAG_GRID=148 timeout 600 python tools/trace_factor.py --n 10000 --nb 128 --ib 16 --out $OUT/trace148.json > $OUT/trace148.log 2>&1
python tools/trace_sm.py $OUT/trace148.json > $OUT/trace148_sm.txt 2>&1; rm -f $OUT/trace148.json
timeout 600 python tools/trace_factor.py --n 10000 --nb 128 --ib 16 --out $OUT/trace.json > $OUT/trace.log 2>&1
python tools/trace_sm.py $OUT/trace.json > $OUT/trace_sm.txt 2>&1; rm -f $OUT/trace.json
echo done
