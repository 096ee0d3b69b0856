#!/bin/bash
# session 4: evidence after the one-CTA-per-SM rule for small DAGs
OUT=gpurun_out/r02s4d
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/t_all.log 2>&1; echo "rc=$?" >> $OUT/t_all.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py --workload 2 --steps 20 --no-cpu-baseline > $OUT/bench_w2.json 2> $OUT/bench_w2.err
timeout 600 python bench.py --workload 0 --steps 20 --no-cpu-baseline > $OUT/bench_w0.json 2> $OUT/bench_w0.err
timeout 900 python bench.py > $OUT/bench_w3.json 2> $OUT/bench_w3.err; echo "rc=$?" >> $OUT/bench_w3.err
for thr in 0 1200; do
  printf "thr=%s " $thr >> $OUT/ab.log
  TILEQR_DAG_ONE_CTA_TILES=$thr python tools/perf_scan.py --n 2048 --pairs 64:16,64:32,96:16,128:16 2>/dev/null | cut -c1-90 | tr '\n' ' ' >> $OUT/ab.log
  echo >> $OUT/ab.log
done
tail -3 $OUT/t_all.log; tail -2 $OUT/smoke.log; cut -c1-200 $OUT/bench_w2.json; cut -c1-200 $OUT/bench_w0.json; cut -c1-200 $OUT/bench_w3.json; cat $OUT/ab.log
