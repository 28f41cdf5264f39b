#!/bin/bash
# Timing bound of the dynamic fused kernel without dependency waits (CHEB_FUSED_NOWAIT: wrong
# results, diagnostic only) next to the real one.
for NW in 0 1; do
  if [ $NW = 1 ]; then export CHEB_FUSED_NOWAIT=1; else unset CHEB_FUSED_NOWAIT; fi
  CHEB_FUSION=3 CHEB_FUSED_LAG=${LAG:-0.5} timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,smsp__inst_executed.sum --clock-control none -k regex:cheb_step2 -s 5 -c 2 --csv python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 1 > gpurun_out/sweep_nw${NW}.csv 2>/dev/null
done
