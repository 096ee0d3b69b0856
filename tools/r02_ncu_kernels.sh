#!/bin/bash
# Round-2 kernel evidence (one gpurun call, ncu only): update_v2_kernel on
# configs[1] 4096-pair batches, layout kernels at 10000^2, batched panel kernels.
OUT=gpurun_out/r02_ncu
mkdir -p $OUT
K="python tools/kernel_cases.py"
run() {  # name, regex, skip, count, cmd...
  local name=$1 re=$2 s=$3 c=$4; shift 4
  if timeout 300 "$@" > $OUT/$name.plain.log 2>&1; then
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$re" -s $s -c $c \
      -o $OUT/$name -f "$@" > $OUT/$name.ncu.log 2>&1
    echo "$name ncu rc=$?" >> $OUT/status.txt
    # bring back text only (the 64 MiB gpurun_out limit): raw counters + per-line source view
    ncu -i $OUT/$name.ncu-rep --page raw --csv > $OUT/$name.raw.csv 2>/dev/null
    ncu -i $OUT/$name.ncu-rep --page source --csv > $OUT/$name.source.csv 2>/dev/null
    gzip -f $OUT/$name.source.csv
    [ "${KEEP_REP:-0}" = "1" ] || rm -f $OUT/$name.ncu-rep
  else
    echo "$name plain run failed" >> $OUT/status.txt
  fi
}
run ssrfb_nb128_ib16 update_v2_kernel 1 1 $K ssrfb 128 16
run ssrfb_nb256_ib32 update_v2_kernel 1 1 $K ssrfb 256 32
run layout_n10000_nb128 "layout_to_tiles|tiles_to_layout" 0 2 $K layout 10000 128 16
run tsqrt_nb128_ib16_b148 panel_fast_kernel 1 1 $K panel tsqrt 128 16 --batch 148
run geqrt_nb128_ib16_b148 panel_fast_kernel 1 1 $K panel geqrt 128 16 --batch 148
