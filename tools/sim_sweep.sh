#!/bin/bash
# Sweep the claim-order simulation's durations (TILEQR_DAG_SIM=sT,sG,hand ns)
# at 10000^2 NB=128; one process per setting (the item list is built once).
for ib in ${IBS:-16 32}; do
for s in ${SIMS:-3000,5000,5000 3000,3000,5000 2500,3000,3000 3000,3500,5000 2000,2500,5000 3000,3000,8000}; do
  printf "%s ib=%s " "$s" "$ib"
  TILEQR_DAG_SIM=$s python tools/perf_scan.py --n ${N:-10000} --pairs 128:$ib
done
done
