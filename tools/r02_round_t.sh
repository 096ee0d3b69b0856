#!/bin/bash
OUT=gpurun_out/r02t
mkdir -p $OUT
timeout 600 python tools/critical_path.py --n 2048 --nb 64 --ib 16 > $OUT/cp2048.log 2>&1
timeout 600 python tools/critical_path.py --n 10000 --nb 128 --ib 16 > $OUT/cp10000.log 2>&1
timeout 2400 python tools/autotune.py --n 20000 40000 --es 0 --out $OUT/tune_big.json --table $OUT/table_big.json > $OUT/autotune_big.log 2>&1; echo "rc=$?" >> $OUT/autotune_big.log
