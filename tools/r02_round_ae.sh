#!/bin/bash
# full GPU suite + smoke + bench lines after the panel-step / sub-task changes
OUT=gpurun_out/r02ae
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > $OUT/t_all.log 2>&1; echo "rc=$?" >> $OUT/t_all.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_w3.json 2> $OUT/bench_w3.err; echo "rc=$?" >> $OUT/bench_w3.err
timeout 600 python bench.py --workload 2 --steps 20 > $OUT/bench_w2.json 2> $OUT/bench_w2.err
for r in 1 2; do for sc in 16 8; do echo "== sc$sc"; TILEQR_PANEL_SUB=$sc python tools/perf_scan.py --n 1024 2048 --pairs 64:8,32:8; done; done > $OUT/sc8.log 2>&1
