#!/bin/bash
# Timed prof_step runs of configs[3] for tuning builds under build_variants/ (and the default
# build), doubling on/off.  Usage on the GPU box: VARIANTS="dbl4 dbl4u4" bash scripts/sweep_variants.sh
for V in default ${VARIANTS}; do
  LIB=""; [ "$V" != default ] && LIB=build_variants/libchebld_$V.so
  for D in ${DBL_LIST:-0 1}; do
    CHEB_LIB=$LIB CHEB_DOUBLING=$D timeout 300 python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 3 > gpurun_out/var_${V}_d${D}.txt 2>&1
    CHEB_LIB=$LIB CHEB_DOUBLING=$D timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,smsp__inst_executed.sum --clock-control none -k regex:cheb_step_kernel -s 10 -c 3 --csv python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 1 > gpurun_out/sweep_${V}_d${D}.csv 2>/dev/null
  done
done
