#!/bin/bash
# GPU call: full GPU suite after the reflector-scaling fix and the wide panels; bench; 2048^2 scan
OUT=gpurun_out/r02j
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $OUT/t_all.log 2>&1; echo "rc=$?" >> $OUT/t_all.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
python tools/perf_scan.py --n 2048 --pairs 64:64,96:48,128:64,160:40,192:48,192:64,256:64,224:56,64:16,128:16 > $OUT/scan.log 2>&1
python tools/perf_scan.py --panel --n --pairs 128:16,64:16,128:64,64:64 > $OUT/panel.log 2>&1
