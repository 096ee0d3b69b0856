#!/bin/bash
# IB through lcm(IB, 8) (R23) + live launch timing in bench: new tests, parity subset,
# bench line, Step-1 and 2048^2 rates of the lcm pairs against base (HEAD)
OUT=gpurun_out/r02an
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_ib_lcm.py tests/test_gpu_factor.py tests/test_gpu_kernels.py tests/test_gpu_tune.py -x -q -p no:cacheprovider > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench_w3.json 2> $OUT/bench_w3.err
B=paper_1102_5328_b200/libtileqr_base.so
P=64:2,128:4,96:12,192:6,160:10,160:20,224:28,224:14,256:1
for v in new base; do
  if [ $v = new ]; then L=paper_1102_5328_b200/libtileqr.so; else L=$B; fi
  echo "== $v"
  TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --n 2048 --pairs $P
  TILEQR_LIB=$L timeout 300 python tools/perf_scan.py --ssrfb --pairs 160:10,160:20,96:12,128:4,64:2
done > $OUT/ab.log 2>&1
echo done
