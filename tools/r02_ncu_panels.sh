#!/bin/bash
# ncu source-level captures of the batched panel kernels (current code)
OUT=gpurun_out/r02_ncu2
mkdir -p $OUT
K="python tools/kernel_cases.py"
run() {  # name, regex, skip, count, cmd...
  local name=$1 re=$2 s=$3 c=$4; shift 4
  if timeout 300 "$@" > $OUT/$name.plain.log 2>&1; then
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$re" -s $s -c $c \
      -o $OUT/$name -f "$@" > $OUT/$name.ncu.log 2>&1
    echo "$name ncu rc=$?" >> $OUT/status.txt
    ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/$name.raw.csv 2>/dev/null
    ncu -i $OUT/$name.ncu-rep --page source --csv > $OUT/$name.source.csv 2>/dev/null
    gzip -f $OUT/$name.source.csv
    rm -f $OUT/$name.ncu-rep
  else
    echo "$name plain run failed" >> $OUT/status.txt
  fi
}
run geqrt_nb128_ib16_b148 panel_fast_kernel 1 1 $K panel geqrt 128 16 --batch 148
run tsqrt_nb128_ib16_b148 panel_fast_kernel 1 1 $K panel tsqrt 128 16 --batch 148
run geqrt_nb64_ib16_b148 panel_fast_kernel 1 1 $K panel geqrt 64 16 --batch 148
