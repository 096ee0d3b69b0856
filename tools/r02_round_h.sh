#!/bin/bash
# GPU call: kernel + factor tests (wide packed panels, scaled inputs, two streams), tree tests,
# Step-1 rates of the configs[1] grid.
OUT=gpurun_out/r02h
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_factor.py tests/test_gpu_parity.py tests/test_gpu_tree.py -x -q -p no:cacheprovider > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
python tools/perf_scan.py --n 2048 --ssrfb --pairs 64:64,96:48,128:64,160:40,192:48,128:16,96:16,160:16,192:16,64:16 > $OUT/scan.log 2>&1
