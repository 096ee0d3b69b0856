#!/bin/bash
# GPU call: host-pipeline tests after the STORE-group change, full bench, ncu launch list and one
# full capture of the dataflow kernel (text exports only; the .ncu-rep stays on the box).
OUT=gpurun_out/r02e
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_factor.py -x -q -p no:cacheprovider -k "host or dataflow" > $OUT/t_host.log 2>&1; echo "rc=$?" >> $OUT/t_host.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "rc=$?" >> $OUT/bench.err
BCMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
if timeout 300 $BCMD > $OUT/bench_short.json 2>&1; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv $BCMD > $OUT/ncu_launch.log 2>&1
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:dag_kernel -s 3 -c 1 -o $OUT/prof_dag -f $BCMD > $OUT/ncu_full.log 2>&1
  ncu -i $OUT/prof_dag.ncu-rep --page raw --csv > $OUT/prof_dag.raw.csv 2>/dev/null
  ncu -i $OUT/prof_dag.ncu-rep --page source --csv --print-source cuda,sass > $OUT/prof_dag.source.csv 2>/dev/null || ncu -i $OUT/prof_dag.ncu-rep --page source --csv > $OUT/prof_dag.source.csv 2>/dev/null
  gzip -f $OUT/prof_dag.source.csv
  rm -f $OUT/prof_dag.ncu-rep
fi
# claim-granularity experiments (same box): panel sub-task width
for sc in 32 16 64 32; do echo "sub=$sc"; TILEQR_PANEL_SUB=$sc python tools/perf_scan.py --n 10000 --pairs 128:16,128:32; done > $OUT/scan_sub.log 2>&1
