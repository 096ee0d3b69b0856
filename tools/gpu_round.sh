#!/bin/bash
# One GPU measurement round: smoke, bench, ncu launch list, ncu full capture of SSRFB.
set -x
OUT=gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
BCMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $BCMD > $OUT/bench_short.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $OUT/launches.csv $BCMD > $OUT/ncu_launch.log 2>&1
echo "ncu launches rc=$?" >> $OUT/ncu_launch.log
SCMD="python tools/perf_scan.py --ssrfb --n --pairs ${PAIR:-64:16}"
timeout 300 $SCMD > $OUT/scan_short.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dmma_update -s 3 -c 1 -o $OUT/prof_ssrfb -f $SCMD > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $OUT/ncu_full.log
