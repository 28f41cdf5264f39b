#!/bin/bash
# Temporal-fusion sweep on configs[3]: forced pairs (CHEB_FUSION=3) per tuning build; timed
# prof_step runs + ncu time/DRAM bytes of steady-state fused launches.
for V in default ${VARIANTS}; do
  LIB=""; [ "$V" != default ] && LIB=build_variants/libchebld_$V.so
  CHEB_LIB=$LIB CHEB_FUSION=3 CHEB_DEBUG=1 timeout 300 python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 3 > gpurun_out/fvar_${V}.txt 2>&1
  CHEB_LIB=$LIB CHEB_FUSION=3 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,smsp__inst_executed.sum --clock-control none -k regex:cheb_step2_kernel -s 5 -c 2 --csv python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 1 > gpurun_out/sweep_f${V}.csv 2>/dev/null
done
