#!/bin/bash
# Step-kernel schedule sweep on configs[3] (gmrf5000): per-launch time and DRAM bytes for
# doubling on/off x resident CTAs per SM.  Run on the GPU box via gpurun; writes gpurun_out/sweep_*.
for D in ${DBL_LIST:-0 1}; do for O in ${OCC_LIST:-2 3 4}; do
  CHEB_DOUBLING=$D CHEB_STEP_OCC=$O timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,smsp__inst_executed.sum --clock-control none -k regex:cheb_step_kernel -s 10 -c 3 --csv python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 1 > gpurun_out/sweep_d${D}_o${O}.csv 2>/dev/null
  CHEB_DOUBLING=$D CHEB_STEP_OCC=$O timeout 300 python scripts/prof_step.py --workload gmrf5000 --k 64 --reps 3 > gpurun_out/sweep_d${D}_o${O}.txt 2>&1
done; done
