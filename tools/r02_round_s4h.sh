#!/bin/bash
# session 4: final evidence with tail retirement as its own kernel instantiation (DAGs of at most 4000 tile updates per step)
OUT=gpurun_out/r02s4h
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/t_all.log 2>&1; echo "rc=$?" >> $OUT/t_all.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_w3.json 2> $OUT/bench_w3.err; echo "rc=$?" >> $OUT/bench_w3.err
timeout 600 python bench.py --workload 2 --steps 20 --no-cpu-baseline > $OUT/bench_w2.json 2> $OUT/bench_w2.err
for t in 0 4000; do
  printf "retire_max_tiles=%s " $t >> $OUT/ab.log
  (TILEQR_DAG_RETIRE_MAX_TILES=$t python tools/perf_scan.py --n 3000 --pairs 64:16
   TILEQR_DAG_RETIRE_MAX_TILES=$t python tools/perf_scan.py --n 4000 --pairs 64:16,64:32
   TILEQR_DAG_RETIRE_MAX_TILES=$t python tools/perf_scan.py --n 6000 --pairs 128:16
   TILEQR_DAG_RETIRE_MAX_TILES=$t python tools/perf_scan.py --n 8000 --pairs 128:16
   TILEQR_DAG_RETIRE_MAX_TILES=$t python tools/perf_scan.py --n 10000 --pairs 128:16) 2>/dev/null | cut -c7-80 | tr '\n' ' ' >> $OUT/ab.log
  echo >> $OUT/ab.log
done
tail -3 $OUT/t_all.log; tail -2 $OUT/smoke.log; cut -c1-200 $OUT/bench_w3.json; cut -c1-200 $OUT/bench_w2.json; cat $OUT/ab.log
