#!/bin/bash
# Probe-block size on configs[3] (m = 128): k = 32, 64, 128 for Algorithm 1 and doubling.
for KK in 32 64 128; do
  timeout 300 python scripts/prof_step.py --workload gmrf5000 --k $KK --reps 2 > gpurun_out/var_k${KK}_d0.txt 2>&1
  CHEB_DOUBLING=1 timeout 300 python scripts/prof_step.py --workload gmrf5000 --k $KK --reps 2 > gpurun_out/var_k${KK}_d1.txt 2>&1
done
