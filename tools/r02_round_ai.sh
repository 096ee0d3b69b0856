#!/bin/bash
# per-SM trace of the 10000^2 (128, 16) factorization (tagged claims), 2 CTAs/SM and 1 CTA/SM
OUT=gpurun_out/r02ai
mkdir -p $OUT
timeout 600 python tools/trace_factor.py --n 10000 --nb 128 --ib 16 --out $OUT/trace.json > $OUT/trace.log 2>&1
python tools/trace_sm.py $OUT/trace.json > $OUT/trace_sm.txt 2>&1
TILEQR_DAG_GRID=148 timeout 600 python tools/trace_factor.py --n 10000 --nb 128 --ib 16 --out $OUT/trace148.json > $OUT/trace148.log 2>&1
python tools/trace_sm.py $OUT/trace148.json > $OUT/trace148_sm.txt 2>&1
rm -f $OUT/trace148.json
gzip -f $OUT/trace.json
echo done
