#!/bin/bash
OUT=gpurun_out/r02s
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k config4 > $OUT/t40k.log 2>&1; echo "rc=$?" >> $OUT/t40k.log
timeout 1200 python tools/perf_scan.py --n 40000 --pairs 128:16,160:16,192:16,256:32,256:16 > $OUT/scan40k.log 2>&1
timeout 1500 python tools/perf_dist_emul.py --n 20000 --nb 160 --ib 16 --ranks 2,4,8 > $OUT/emul20k.log 2>&1
