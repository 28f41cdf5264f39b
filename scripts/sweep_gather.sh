#!/bin/bash
# Gather-staged step kernel (CHEB_GATHER=1) vs the regular per-step kernel on configs[3] / [2].
for W in ${WORKLOADS:-gmrf5000}; do
  for GS in 0 1; do
    CHEB_GATHER=$GS CHEB_DEBUG=1 timeout 300 python scripts/prof_step.py --workload $W --k 64 --reps 3 > gpurun_out/var_${W}_gs${GS}.txt 2>&1
    CHEB_GATHER=$GS timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,smsp__inst_executed.sum --clock-control none -k regex:"cheb_step" -s 10 -c 2 --csv python scripts/prof_step.py --workload $W --k 64 --reps 1 > gpurun_out/sweep_${W}_gs${GS}.csv 2>/dev/null
  done
done
