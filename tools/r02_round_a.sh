#!/bin/bash
# GPU call: full GPU test suite, smoke, bench (N=1), autotune over the paper's N grid.
OUT=gpurun_out/r02a
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=20 > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 2400 python tools/autotune.py --out $OUT/tune_r02.json --table $OUT/tuned_table.json > $OUT/autotune.log 2>&1; echo "autotune rc=$?" >> $OUT/autotune.log
