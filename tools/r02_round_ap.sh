#!/bin/bash
# R23 for IB > 64 too: tests, then the 2048^2 tuner run + exhaustive search over the 74-pair grid
OUT=gpurun_out/r02ap
mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_ib_lcm.py tests/test_gpu_factor.py tests/test_gpu_kernels.py tests/test_gpu_tune.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
timeout 1500 python tools/autotune.py --n 2048 --es 2048 --out $OUT/tune_2048_es.json --table $OUT/table_2048.json > $OUT/autotune.log 2>&1; echo "rc=$?" >> $OUT/autotune.log
echo done
