#!/bin/bash
# Fused pairs on gather-staged tiles (CHEB_FUSION=3 + CHEB_GATHER=1: cheb_step2g_kernel) vs the
# warp-specialised fused kernel on regular tiles and vs per-step launches, configs[3] k=64.
W=${WORKLOAD:-gmrf5000}
for CFG in "1 0" "3 0" "3 1"; do
  set -- $CFG; FU=$1; GS=$2
  for LAG in ${LAGS:-1.5}; do
    CHEB_FUSION=$FU CHEB_GATHER=$GS CHEB_FUSED_LAG=$LAG CHEB_DEBUG=1 timeout 300 python scripts/prof_step.py --workload $W --k 64 --reps 3 > gpurun_out/fg_${W}_f${FU}_g${GS}_l${LAG}.txt 2>&1
    CHEB_FUSION=$FU CHEB_GATHER=$GS CHEB_FUSED_LAG=$LAG timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,smsp__inst_executed.sum --clock-control none -k regex:"cheb_step" -s 10 -c 2 --csv python scripts/prof_step.py --workload $W --k 64 --reps 1 > gpurun_out/fgncu_${W}_f${FU}_g${GS}_l${LAG}.csv 2>/dev/null
  done
done
