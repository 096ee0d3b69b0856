#!/bin/bash
# GPU call: bench lines for configs[0], [2], [3] (default), the reference arm, and the
# tuner reliability study on and off the decision table's N grid.
OUT=gpurun_out/r02d
mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_w3.json 2> $OUT/bench_w3.err; echo "rc=$?" >> $OUT/bench_w3.err
timeout 600 python bench.py --workload 0 --steps 20 > $OUT/bench_w0.json 2> $OUT/bench_w0.err; echo "rc=$?" >> $OUT/bench_w0.err
timeout 600 python bench.py --workload 2 --steps 20 > $OUT/bench_w2.json 2> $OUT/bench_w2.err; echo "rc=$?" >> $OUT/bench_w2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 2700 python tools/reliability.py --n 1000 1500 2000 3000 4000 5000 --table paper_1102_5328_b200/tuned_table.json --out $OUT/reliability.json > $OUT/reliability.log 2>&1; echo "rc=$?" >> $OUT/reliability.log
