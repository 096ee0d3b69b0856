#!/bin/bash
# One GPU measurement round (run under gpurun from the repo root):
#   GPU tests, smoke, autotune (optional), bench, ncu launch list, ncu full capture of the dataflow kernel.
# Writes everything under gpurun_out/.
OUT=gpurun_out
R=${ROUND:-r01}
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/gpu_tests.log 2>&1; echo "rc=$?" >> $OUT/gpu_tests.log
fi
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
if [ "${TUNE:-0}" = "1" ]; then
  timeout 1700 python tools/autotune.py > $OUT/autotune.log 2>&1 && cp $OUT/tuned_table.json paper_1102_5328_b200/tuned_table.json
fi
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
BCMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 300 $BCMD > $OUT/bench_short.json 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file $OUT/launches.csv $BCMD > $OUT/ncu_launch.log 2>&1
  echo "ncu launches rc=$?" >> $OUT/ncu_launch.log
  # the dataflow kernel (one launch = the whole factorization): the 4th launch, after the 3 warm-up steps
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dag_kernel -s 3 -c 1 -o $OUT/prof_dag_bench -f $BCMD > $OUT/ncu_full.log 2>&1
  echo "ncu full rc=$?" >> $OUT/ncu_full.log
fi
