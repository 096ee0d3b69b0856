#!/bin/bash
# single-warp panel factorization A/B (libtileqr.so = SW, libtileqr_nosw.so = -DTILEQR_NO_SW_FACTOR)
OUT=gpurun_out/r02v
mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_factor.py tests/test_gpu_tree.py -x -q -p no:cacheprovider -k "not config3 and not config4" > $OUT/t.log 2>&1; echo "rc=$?" >> $OUT/t.log
for r in 1 2 3; do
  echo "sw"; python tools/perf_scan.py --n 1024 2048 4096 --pairs 64:16,96:16,64:8,128:8,32:16 ; python tools/perf_scan.py --n 10000 --pairs 128:16,96:16 ; python tools/perf_scan.py --panel --n --pairs 64:16,96:16,128:8
  echo "nosw"; TILEQR_LIB=paper_1102_5328_b200/libtileqr_nosw.so python tools/perf_scan.py --n 1024 2048 4096 --pairs 64:16,96:16,64:8,128:8,32:16; TILEQR_LIB=paper_1102_5328_b200/libtileqr_nosw.so python tools/perf_scan.py --n 10000 --pairs 128:16,96:16; TILEQR_LIB=paper_1102_5328_b200/libtileqr_nosw.so python tools/perf_scan.py --panel --n --pairs 64:16,96:16,128:8
done > $OUT/ab.log 2>&1
echo done
