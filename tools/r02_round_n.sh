#!/bin/bash
# GPU call: C2-prefetch A/B (same box) + dataflow correctness tests with the new default library
OUT=gpurun_out/r02n
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_factor.py tests/test_gpu_parity.py tests/test_gpu_tree.py tests/test_gpu_dist.py -x -q -p no:cacheprovider > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
for r in 1 2 3; do
  echo "c2pf"; python tools/perf_scan.py --n 10000 4096 --pairs 128:16,128:32,64:16
  echo "noc2pf"; TILEQR_LIB=paper_1102_5328_b200/libtileqr_noc2pf.so python tools/perf_scan.py --n 10000 4096 --pairs 128:16,128:32,64:16
done > $OUT/ab.log 2>&1
