#!/bin/bash
# 8-warp / MB=1 variant (w8): per-item duration quantiles at 10000^2 (128, 16); where (128, 32) hangs
OUT=gpurun_out/r02ar
mkdir -p $OUT
W=paper_1102_5328_b200/libtileqr_w8.so
TILEQR_LIB=$W timeout 300 python tools/trace_factor.py --n 10000 --nb 128 --ib 16 --out $OUT/trace_w8.json > $OUT/trace_w8.log 2>&1
python tools/trace_sm.py $OUT/trace_w8.json > $OUT/trace_w8_sm.txt 2>&1; rm -f $OUT/trace_w8.json
for n in 512 1024 2048 4096; do
  for ib in 32 16; do
    echo "== n=$n ib=$ib" >> $OUT/hang.log
    TILEQR_LIB=$W timeout 60 python tools/perf_scan.py --n $n --pairs 128:$ib >> $OUT/hang.log 2>&1; echo "rc=$?" >> $OUT/hang.log
    TILEQR_SCHED=levels TILEQR_LIB=$W timeout 60 python tools/perf_scan.py --n $n --pairs 128:$ib >> $OUT/hang.log 2>&1; echo "levels rc=$?" >> $OUT/hang.log
  done
done
echo done
