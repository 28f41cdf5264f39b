#!/bin/bash
# k = 128 (one block for m = 128) vs k = 64 on configs[3], builds x schedule.
for V in default ${VARIANTS}; do
  LIB=""; [ "$V" != default ] && LIB=build_variants/libchebld_$V.so
  for KK in 64 128; do
    CHEB_LIB=$LIB timeout 300 python scripts/prof_step.py --workload gmrf5000 --k $KK --reps 3 > gpurun_out/var_${V}_k${KK}.txt 2>&1
    CHEB_LIB=$LIB CHEB_DOUBLING=1 timeout 300 python scripts/prof_step.py --workload gmrf5000 --k $KK --reps 3 > gpurun_out/var_${V}_k${KK}_dbl.txt 2>&1
  done
done
