#!/bin/bash
# Warp-specialised fused pairs on configs[3]: builds x lag (CHEB_FUSION=3).
for V in default ${VARIANTS}; do
  LIB=""; [ "$V" != default ] && LIB=build_variants/libchebld_$V.so
  for LAG in ${LAGS:-1 1.5 2}; do
    CHEB_LIB=$LIB CHEB_FUSION=3 CHEB_FUSED_LAG=$LAG timeout 300 python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 3 > gpurun_out/var_${V}_l${LAG}.txt 2>&1
    CHEB_LIB=$LIB CHEB_FUSION=3 CHEB_FUSED_LAG=$LAG timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,smsp__inst_executed.sum --clock-control none -k regex:cheb_step2 -s 5 -c 2 --csv python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 1 > gpurun_out/sweep_${V}_l${LAG}.csv 2>/dev/null
  done
done
