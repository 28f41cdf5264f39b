#!/bin/bash
# L2 prefetch of first-touch gather rows: default build (on) vs pf0 (off), per schedule.
for V in default pf1; do
  LIB=""; [ "$V" != default ] && LIB=build_variants/libchebld_$V.so
  for S in d0 d1 f3; do
    ENV=""; KR=cheb_step_kernel
    [ $S = d1 ] && ENV="CHEB_DOUBLING=1"
    [ $S = f3 ] && ENV="CHEB_FUSION=3" && KR=cheb_step2
    env CHEB_LIB=$LIB $ENV timeout 300 python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 3 > gpurun_out/var_${V}_${S}.txt 2>&1
    env CHEB_LIB=$LIB $ENV timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,smsp__inst_executed.sum --clock-control none -k regex:$KR -s 10 -c 2 --csv python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 1 > gpurun_out/sweep_${V}_${S}.csv 2>/dev/null
  done
done
