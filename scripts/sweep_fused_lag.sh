#!/bin/bash
# Dynamic-ticket fused pairs on configs[3]: lag sweep (CHEB_FUSED_LAG waves beyond the halo).
for LAG in ${LAGS:-0.5 1 1.5}; do
  CHEB_FUSION=3 CHEB_FUSED_LAG=$LAG CHEB_DEBUG=1 timeout 300 python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 3 > gpurun_out/var_lag${LAG}.txt 2>&1
  CHEB_FUSION=3 CHEB_FUSED_LAG=$LAG timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,smsp__inst_executed.sum --clock-control none -k regex:cheb_step2 -s 5 -c 2 --csv python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 1 > gpurun_out/sweep_lag${LAG}.csv 2>/dev/null
done
