#!/bin/bash
# Persistent kernel (L2-resident operators): grid size sweep via CHEB_MIN_TILES on configs 0/1.
for W in ${WORKLOADS:-torus256 gmrf32}; do
  for MT in ${MTS:-1 2 4 8}; do
    CHEB_MIN_TILES=$MT timeout 300 python scripts/prof_step.py --workload $W --reps 3 --k ${K:-0} > gpurun_out/var_${W}_mt${MT}.txt 2>&1
    CHEB_DOUBLING=1 CHEB_MIN_TILES=$MT timeout 300 python scripts/prof_step.py --workload $W --reps 3 --k ${K:-0} > gpurun_out/var_${W}_mt${MT}_dbl.txt 2>&1
  done
done
