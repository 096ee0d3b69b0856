#!/bin/bash
# final evidence of the session: full GPU suite, smoke, bench lines (configs[3], [2], [0], tall-skinny tree),
# reference arm, ncu launch list and one full capture of the dataflow kernel
OUT=gpurun_out/r02fin2
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/t_all.log 2>&1; echo "rc=$?" >> $OUT/t_all.log
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 900 python bench.py > $OUT/bench_w3.json 2> $OUT/bench_w3.err; echo "rc=$?" >> $OUT/bench_w3.err
timeout 600 python bench.py --workload 2 --steps 20 --no-cpu-baseline > $OUT/bench_w2.json 2> $OUT/bench_w2.err
timeout 600 python bench.py --workload 0 --steps 20 --no-cpu-baseline > $OUT/bench_w0.json 2> $OUT/bench_w0.err
timeout 600 python bench.py --workload 5 > $OUT/bench_w5.json 2> $OUT/bench_w5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
BCMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 300 $BCMD > $OUT/bench_short.json 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $OUT/launches.csv $BCMD > $OUT/ncu_launch.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dag_kernel -s 3 -c 1 -o $OUT/prof_dag -f $BCMD > $OUT/ncu_full.log 2>&1
  ncu -i $OUT/prof_dag.ncu-rep --page raw --csv > $OUT/prof_dag.raw.csv 2>/dev/null
  ncu -i $OUT/prof_dag.ncu-rep --page source --csv > $OUT/prof_dag.source.csv 2>/dev/null
  gzip -f $OUT/prof_dag.source.csv; rm -f $OUT/prof_dag.ncu-rep
fi
echo done
