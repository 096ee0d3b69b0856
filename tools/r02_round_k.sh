#!/bin/bash
# GPU call: refreshed Step 1 + exhaustive search at 2048 (wide panels), the tall-skinny bench line,
# ncu of the new layout kernels and of the wide packed update.
OUT=gpurun_out/r02k
mkdir -p $OUT
timeout 1200 python tools/autotune.py --n 2048 --es 2048 --out $OUT/tune_2048.json --table $OUT/table_2048.json > $OUT/autotune.log 2>&1; echo "rc=$?" >> $OUT/autotune.log
timeout 900 python bench.py --workload 5 > $OUT/bench_w5.json 2> $OUT/bench_w5.err; echo "rc=$?" >> $OUT/bench_w5.err
K="python tools/kernel_cases.py"
prof() {  # name regex skip count cmd...
  local name=$1 re=$2 s=$3 c=$4; shift 4
  if timeout 300 "$@" > $OUT/$name.plain.log 2>&1; then
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$re" -s $s -c $c -o $OUT/$name -f "$@" > $OUT/$name.ncu.log 2>&1
    ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/$name.raw.csv 2>/dev/null
    rm -f $OUT/$name.ncu-rep
  fi
}
prof layout2_n10000_nb128 "layout_to_tiles|tiles_to_layout" 0 2 $K layout 10000 128 16
prof ssrfb_wide_nb128_ib64 update_v2_kernel 1 1 $K ssrfb 128 64
prof ssrfb_wide_nb192_ib48 update_v2_kernel 1 1 $K ssrfb 192 48
python tools/perf_scan.py --panel --n --pairs 128:16,128:64,64:64,192:48 > $OUT/panel.log 2>&1
python tools/perf_scan.py --n 2048 --pairs 64:64,96:48,128:64,160:40,192:48,256:64 > $OUT/scan.log 2>&1
